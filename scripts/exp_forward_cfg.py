"""Time K2 at C2 and C5 shapes for a few launch geometries, interleaved and repeated (tuning check)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2504_08339_b200 as fnb  # noqa: E402
from paper_2504_08339_b200.synthetic import regression_dataset, synthetic_population  # noqa: E402

cfgs = json.loads(sys.argv[1])  # [[cols, rows_pct, recs_pct, kb], ...]
dev = torch.device("cuda", 0)
lib = fnb._native.lib()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
X_h, Y_h = regression_dataset(1024, 4, 1, seed=0)
X = torch.from_numpy(X_h.astype(np.float32)).to(dev)
Y = torch.from_numpy(Y_h.astype(np.float32)).to(dev)
out = {}
for name, (P, N, C) in {"c2": (10_000, 64, 256), "c5": (20_000, 128, 1024)}.items():
    n_h, c_h = synthetic_population(P, N, C, 0.75, 4, 1, seed=1000)
    eng = fnb.Engine(fnb.GenomeLimits(N, C), [0, 1, 2, 3], [4], fnb.AttributeSchema())
    nodes, conns = torch.from_numpy(n_h).to(dev), torch.from_numpy(c_h).to(dev)
    nets = eng.alloc_nets(P)
    st = torch.cuda.current_stream()
    eng.transform_d(nodes, conns, nets, st)
    fit = torch.empty(P, dtype=torch.float64, device=dev)
    res = {i: [] for i in range(len(cfgs))}
    for rep in range(5):
        for i, (cols, pct, rp, kb) in enumerate(cfgs):
            lib.fnb_set_forward_tuning(2, cols, pct, kb)
            lib.fnb_set_forward_recs_pct(rp)
            eng.forward_d(nets, P, X, Y, fnb.FIT_NEG_MSE, 0.0, fitness=fit, stream=st)
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            eng.forward_d(nets, P, X, Y, fnb.FIT_NEG_MSE, 0.0, fitness=fit, stream=st)
            b.record(st)
            torch.cuda.synchronize()
            res[i].append(a.elapsed_time(b))
    out[name] = {str(cfgs[i]): [round(float(np.median(v)), 4), round(float(np.min(v)), 4), round(float(np.max(v)), 4)]
                 for i, v in res.items()}
    del nodes, conns, nets
print(json.dumps(out, indent=1))
