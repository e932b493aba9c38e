"""Distribution of K1's per-genome value-slot and record counts (NetHeader) on the bench populations."""
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
from paper_2504_08339_b200.synthetic import synthetic_population  # noqa: E402

dev = torch.device("cuda", 0)
out = {}
for name, (P, N, C) in {"c2": (10_000, 64, 256), "c5": (20_000, 128, 1024)}.items():
    n_h, c_h = synthetic_population(P, N, C, 0.75, 4, 1, seed=1000)
    eng = fnb.Engine(fnb.GenomeLimits(N, C), [0, 1, 2, 3], [4], fnb.AttributeSchema())
    nets = eng.alloc_nets(P)
    eng.transform_d(torch.from_numpy(n_h).to(dev), torch.from_numpy(c_h).to(dev), nets, torch.cuda.current_stream())
    torch.cuda.synchronize()
    hb = nets.view(P, -1)[:, :32].cpu().numpy()
    h = hb.view(np.int32).reshape(P, 8)
    h16 = hb.view(np.int16).reshape(P, 16)
    n_slots = h[:, 6]
    if os.environ.get("FNB_DUMP_SLOTS"):
        np.save(os.environ["FNB_DUMP_SLOTS"] + f"_{name}.npy", n_slots)
    n_rec = h16[:, 11]
    n_ops = h16[:, 9]
    n_edges = h16[:, 10]
    q = [0, 10, 25, 50, 75, 90, 99, 100]
    out[name] = {"n_slots_pct": dict(zip(q, np.percentile(n_slots, q).tolist())),
                 "n_rec_pct": dict(zip(q, np.percentile(n_rec, q).tolist())),
                 "mean_slots": float(n_slots.mean()), "mean_rec": float(n_rec.mean()),
                 "mean_ops": float(n_ops.mean()), "mean_edges": float(n_edges.mean())}
print(json.dumps(out, indent=1))
