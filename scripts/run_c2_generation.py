"""The C2 device generation loop alone (profiling driver): pop 10k, N64/C256,
synthetic start population, `G` generations of evaluate + step."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if os.environ.get("FNB_AB_ROOT"):  # A/B: a package copy with another library build
    sys.path.insert(0, os.environ["FNB_AB_ROOT"])
import paper_2504_08339_b200 as fnb  # noqa: E402
from paper_2504_08339_b200.evolve import Evolver, NeatConfig  # noqa: E402
from paper_2504_08339_b200.synthetic import regression_dataset, synthetic_population  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 5
dev = torch.device("cuda", 0)
eng = fnb.Engine(fnb.GenomeLimits(64, 256), [0, 1, 2, 3], [4], fnb.AttributeSchema())
ev = Evolver(eng, NeatConfig(pop_size=10_000), seed=1000)
n, c = synthetic_population(10_000, 64, 256, 0.75, 4, 1, seed=1000)
ev.set_population(n, c)
X_h, Y_h = regression_dataset(1024, 4, 1, seed=0)
X = torch.from_numpy(X_h.astype(np.float32)).to(dev)
Y = torch.from_numpy(Y_h.astype(np.float32)).to(dev)
for _ in range(G):
    ev.evaluate_d(X, Y)
    ev.step()
torch.cuda.synchronize()
print("ok", ev.state(), ev.species()["count"])
