"""Sweep the K2 launch geometry (fnb_set_forward_tuning) on the bench workload.

Every configuration must reproduce the default configuration's fitness bit
for bit (the 32-sample fitness units make the FP64 sums independent of the
geometry); the script asserts that, then prints the fastest configurations.

    python scripts/sweep_forward.py > gpurun_out/sweep.txt
"""
import itertools
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2504_08339_b200 as fnb  # noqa: E402
from paper_2504_08339_b200.synthetic import regression_dataset, synthetic_population  # noqa: E402


def main():
    P, N, C, B, NI, NO = 10_000, 64, 256, 1024, 4, 1
    if os.environ.get("FNB_SWEEP_SHAPE") == "c5":  # C5 genome shapes, 20k genomes (K2 is linear in P)
        P, N, C = 20_000, 128, 1024
    dev = torch.device("cuda", 0)
    nodes_h, conns_h = synthetic_population(P, N, C, 0.75, NI, NO, seed=1000)
    X_h, Y_h = regression_dataset(B, NI, NO, seed=0)
    eng = fnb.Engine(fnb.GenomeLimits(N, C), list(range(NI)), list(range(NI, NI + NO)), fnb.AttributeSchema())
    nodes, conns = torch.from_numpy(nodes_h).to(dev), torch.from_numpy(conns_h).to(dev)
    X = torch.from_numpy(X_h.astype(np.float32)).to(dev)
    Y = torch.from_numpy(Y_h.astype(np.float32)).to(dev)
    nets = eng.alloc_nets(P)
    st = torch.cuda.current_stream()
    eng.transform_d(nodes, conns, nets, st)
    fit = torch.empty(P, dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    lib = fnb._native.lib()

    def run(reps=10):
        eng.forward_d(nets, P, X, Y, fnb.FIT_NEG_MSE, 0.0, fitness=fit, stream=st)
        ms = []
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            eng.forward_d(nets, P, X, Y, fnb.FIT_NEG_MSE, 0.0, fitness=fit, stream=st)
            b.record(st)
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        return float(np.median(ms))

    lib.fnb_set_forward_tuning(0, 0, 0, 0)
    base_ms = run()
    base_fit = fit.clone()
    res = []
    grid = ((2, 4), (128, 256, 512), (45, 50, 55, 62, 75), (72,))
    recs_grid = (40, 50, 60, 75, 100)
    if os.environ.get("FNB_SWEEP_GRID"):  # JSON [[spt...], [cols...], [pct...], [kb...], [recs_pct...]]
        g = json.loads(os.environ["FNB_SWEEP_GRID"])
        grid, recs_grid = tuple(tuple(x) for x in g[:4]), tuple(g[4])
    if os.environ.get("FNB_SWEEP_SHAPE") == "c5":
        grid = ((2, 4), (64, 128, 256), (30, 40, 50, 62, 75), (72, 144))
    for spt, cols, pct, kb, rp in itertools.product(*grid, recs_grid):
        lib.fnb_set_forward_tuning(spt, cols, pct, kb)
        lib.fnb_set_forward_recs_pct(rp)
        try:
            ms = run()
        except Exception as e:  # geometry that does not fit is reported, not fatal
            res.append({"spt": spt, "cols": cols, "pct": pct, "kb": kb, "recs_pct": rp, "error": str(e)[:80]})
            continue
        same = bool(torch.equal(fit, base_fit))
        res.append({"spt": spt, "cols": cols, "pct": pct, "kb": kb, "recs_pct": rp, "ms": ms, "bit_equal": same})
        assert same, ("fitness bits changed with the launch geometry", spt, cols, pct, kb, rp)
    lib.fnb_set_forward_tuning(0, 0, 0, 0)
    lib.fnb_set_forward_recs_pct(0)
    ok = sorted([r for r in res if "ms" in r], key=lambda r: r["ms"])
    best_by_spt = {spt: min((r for r in ok if r["spt"] == spt), key=lambda r: r["ms"], default=None)
                   for spt in (2, 4)}
    print(json.dumps({"default_ms": base_ms, "best": ok[:12], "all": ok, "best_by_spt": best_by_spt,
                      "errors": [r for r in res if "error" in r][:5], "n": len(res)}, indent=1))


if __name__ == "__main__":
    main()
