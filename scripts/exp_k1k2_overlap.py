"""Experiment: overlap K1 (transform) of chunk k+1 with K2 (forward) of chunk k on two streams."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2504_08339_b200 as fnb  # noqa: E402
from paper_2504_08339_b200.synthetic import regression_dataset, synthetic_population  # noqa: E402

P, N, C, B = 10_000, 64, 256, 1024
dev = torch.device("cuda", 0)
n_h, c_h = synthetic_population(P, N, C, 0.75, 4, 1, seed=1000)
X_h, Y_h = regression_dataset(B, 4, 1, seed=0)
eng = fnb.Engine(fnb.GenomeLimits(N, C), [0, 1, 2, 3], [4], fnb.AttributeSchema())
nodes, conns = torch.from_numpy(n_h).to(dev), torch.from_numpy(c_h).to(dev)
X = torch.from_numpy(X_h.astype(np.float32)).to(dev)
Y = torch.from_numpy(Y_h.astype(np.float32)).to(dev)
nets = eng.alloc_nets(P)
nb = eng.net_bytes
fit = torch.empty(P, dtype=torch.float64, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
s0 = torch.cuda.current_stream()
s1 = torch.cuda.Stream()


def run(chunks):
    bounds = [P * k // chunks for k in range(chunks + 1)]
    evs = [torch.cuda.Event() for _ in range(chunks)]
    for k in range(chunks):
        lo, hi = bounds[k], bounds[k + 1]
        eng.transform_d(nodes[lo:hi], conns[lo:hi], nets[lo * nb:hi * nb], s1)
        evs[k].record(s1)
    for k in range(chunks):
        lo, hi = bounds[k], bounds[k + 1]
        s0.wait_event(evs[k])
        eng.forward_d(nets[lo * nb:hi * nb], hi - lo, X, Y, fnb.FIT_NEG_MSE, 0.0, fitness=fit[lo:hi], stream=s0)


def timeit(chunks, reps=20):
    run(chunks)
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s0)
        s1.wait_stream(s0)
        run(chunks)
        s0.wait_stream(s1)
        b.record(s0)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    return float(np.median(ms))


ref = None
for ch in (1, 2, 3, 4, 8):
    t = timeit(ch)
    f = fit.clone()
    if ref is None:
        ref = f
    print(f"chunks {ch}: {t:.4f} ms, fitness bit-equal {bool(torch.equal(f, ref))}")
