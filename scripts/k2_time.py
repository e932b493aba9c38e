"""Time K2 (forward + fitness) on the bench workloads and print a fitness hash.

Run once per variant (environment knobs such as FNB_FWD_CHUNKS / FNB_FWD_SPT
are read by the library at first use); equal hashes = bit-identical fitness.

    python scripts/k2_time.py [c2|c5|c3|rich ...]
"""
import hashlib
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if os.environ.get("FNB_AB_ROOT"):  # A/B: a package copy with another library build
    sys.path.insert(0, os.environ["FNB_AB_ROOT"])
import paper_2504_08339_b200 as fnb  # noqa: E402
from paper_2504_08339_b200.synthetic import regression_dataset, synthetic_population  # noqa: E402

SHAPES = {"c2": (10_000, 64, 256, 1024), "c5": (20_000, 128, 1024, 1024), "c3": (2_000, 64, 256, 65536),
          "rich": (10_000, 64, 256, 1024)}


def main():
    names = sys.argv[1:] or ["c2"]
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out = {"env": {k: v for k, v in os.environ.items() if k.startswith("FNB_")}}
    for name in names:
        P, N, C, B = SHAPES[name]
        rich = name == "rich"
        na, ng = (5, 4) if rich else (1, 1)
        n_h, c_h = synthetic_population(P, N, C, 0.75, 4, 1, n_act=na, n_agg=ng, seed=1000)
        X_h, Y_h = regression_dataset(B, 4, 1, seed=0)
        schema = (fnb.AttributeSchema(["tanh", "sigmoid", "identity", "relu", "sin"], ["sum", "product", "max", "mean"])
                  if rich else fnb.AttributeSchema())
        eng = fnb.Engine(fnb.GenomeLimits(N, C), [0, 1, 2, 3], [4], schema)
        nodes, conns = torch.from_numpy(n_h).to(dev), torch.from_numpy(c_h).to(dev)
        X = torch.from_numpy(X_h.astype(np.float32)).to(dev)
        Y = torch.from_numpy(Y_h.astype(np.float32)).to(dev)
        nets = eng.alloc_nets(P)
        st = torch.cuda.current_stream()
        fit = torch.empty(P, dtype=torch.float64, device=dev)
        k1, k2 = [], []
        for rep in range(12):
            flush.zero_()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            ev[0].record(st)
            eng.transform_d(nodes, conns, nets, st)
            ev[1].record(st)
            eng.forward_d(nets, P, X, Y, fnb.FIT_NEG_MSE, 0.0, fitness=fit, stream=st)
            ev[2].record(st)
            torch.cuda.synchronize()
            if rep >= 2:
                k1.append(ev[0].elapsed_time(ev[1]))
                k2.append(ev[1].elapsed_time(ev[2]))
        h = hashlib.sha256(fit.cpu().numpy().tobytes()).hexdigest()[:16]
        evals = P * B
        out[name] = {"k1_ms": round(float(np.median(k1)), 4), "k2_ms": round(float(np.median(k2)), 4),
                     "k2_min": round(float(np.min(k2)), 4), "gevals": round(evals / np.median(k2) / 1e6, 3),
                     "fit_hash": h}
        del nodes, conns, nets
    print(json.dumps(out))


if __name__ == "__main__":
    main()
