"""BASELINE config 1 as a search problem: XOR (3 inputs incl. bias),
pop 1000, N16/C32, fitness 4 - SSE, target 3.9, at most 100 generations, seeds 0..9,
through fnb_evolve (one CUDA graph per generation)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2504_08339_b200 as fnb  # noqa: E402
from paper_2504_08339_b200.evolve import NeatConfig, evolve  # noqa: E402
from paper_2504_08339_b200.synthetic import xor_dataset  # noqa: E402

eng = fnb.Engine(fnb.GenomeLimits(16, 32), [0, 1, 2], [3], fnb.AttributeSchema(["sigmoid", "tanh"], ["sum"]))
X, Y = xor_dataset(bias_input=True)
solved, gens, times = 0, [], []
for seed in range(10):
    cfg = NeatConfig(pop_size=1000, generation_limit=100, fitness_target=3.9, compatibility_threshold=1.0,
                     output_activation=0)
    t0 = time.perf_counter()
    best, fit, stats = evolve(eng, cfg, seed=seed, X=X, Y=Y, kind=fnb.FIT_OFFSET_SSE, offset=4.0)
    dt = time.perf_counter() - t0
    ok = fit >= 3.9
    solved += ok
    gens.append(len(stats))
    times.append(dt)
    print(f"seed {seed}: {'solved' if ok else 'not solved'} after {len(stats)} generations, best fitness {fit:.4f}, "
          f"species {stats[-1].species_count}, {dt * 1e3:.1f} ms ({dt / len(stats) * 1e3:.2f} ms/generation)")
print(f"solved {solved}/10; generations: mean {np.mean(gens):.1f}, median {np.median(gens):.0f}")
