"""e2e (fnb_evaluate with pinned host buffers) for one H2D chunk size
(FNB_H2D_CHUNK_MB, read by the library at first use).

    for mb in 2 4 8 16; do FNB_H2D_CHUNK_MB=$mb python scripts/sweep_h2d.py; done
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if os.environ.get("FNB_AB_ROOT"):  # A/B: a package copy with another library build
    sys.path.insert(0, os.environ["FNB_AB_ROOT"])
import paper_2504_08339_b200 as fnb  # noqa: E402
from paper_2504_08339_b200.synthetic import regression_dataset, synthetic_population  # noqa: E402

nodes, conns = synthetic_population(10_000, 64, 256, 0.75, 4, 1, seed=1000)
X, Y = regression_dataset(1024, 4, 1, seed=0)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
n, c, x, y = pin(nodes), pin(conns), pin(X), pin(Y)
eng = fnb.Engine(fnb.GenomeLimits(64, 256), [0, 1, 2, 3], [4], fnb.AttributeSchema())
eng.evaluate(n, c, x, y, fnb.FIT_NEG_MSE)
ts = []
for _ in range(20):
    t0 = time.perf_counter()
    eng.evaluate(n, c, x, y, fnb.FIT_NEG_MSE)
    ts.append(time.perf_counter() - t0)
t = float(np.median(ts))
print(json.dumps({"chunk_mb": os.environ.get("FNB_H2D_CHUNK_MB", "8"),
                  "ms": t * 1e3, "gevals": 10_240_000 / t / 1e9, "h2d_gbps": (n.nbytes + c.nbytes) / t / 1e9}))
