"""North-star check at BASELINE config 2 scale: the device generation loop
(pop 10k, N_max=64, C_max=256, B=1024 func-fit, paper defaults) against the
frozen restatement oracle/evolution.c for 100 generations, both sides given
the device's fitness each generation.  The whole evolution
state -- population tensors with their NaN padding, species table, innovation
counter -- is compared bit for bit every generation.

    python scripts/validate_c2_100.py [generations] > profiles/r02_validate_c2_100.txt
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_lib as ol  # noqa: E402
import paper_2504_08339_b200 as fnb  # noqa: E402
from paper_2504_08339_b200.evolve import Evolver, NeatConfig  # noqa: E402
from paper_2504_08339_b200.synthetic import regression_dataset  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 100
P, N, C, B = 10_000, 64, 256, 1024
acts, aggs = ["tanh"], ["sum"]
eng = fnb.Engine(fnb.GenomeLimits(N, C), [0, 1, 2, 3], [4], fnb.AttributeSchema(acts, aggs))
ev = Evolver(eng, NeatConfig(pop_size=P), seed=2025)
orc = ol.OracleEvolution(ol.Problem(N, C, [0, 1, 2, 3], [4]), ol.SchemaSpec(acts, aggs), ol.neat_cfg(P), seed=2025)
ev.init_population()
orc.init_population()
X, Y = regression_dataset(B, 4, 1, seed=0)
t_dev = t_orc = 0.0
for g in range(G):
    t0 = time.perf_counter()
    ev.evaluate(X, Y)
    fit = ev.fitness()
    ev.step()
    t1 = time.perf_counter()
    orc.step(fit)
    t2 = time.perf_counter()
    t_dev += t1 - t0
    t_orc += t2 - t1
    gn, gc = ev.population()
    same_pop = np.array_equal(gn.view(np.uint64), orc.nodes.view(np.uint64)) and \
        np.array_equal(gc.view(np.uint64), orc.conns.view(np.uint64))
    sp, so = ev.species(), orc.species_view()
    same_sp = sp["count"] == so["count"] and all(np.array_equal(sp[k], so[k]) for k in ("ids", "spawn", "best",
                                                                                        "stagnation"))
    same_key = ev.state()[1] == orc.innov.next_key
    n_nodes = float(np.mean(np.sum(~np.isnan(gn[:, :, 0]), axis=1)))
    n_conns = float(np.mean(np.sum(~np.isnan(gc[:, :, 0]), axis=1)))
    print(f"gen {g:3d}: best {fit.max():.6f} species {sp['count']:2d} next_key {ev.state()[1]:6d} "
          f"mean nodes {n_nodes:5.1f} conns {n_conns:6.1f}  population {'==' if same_pop else '!='} "
          f"species {'==' if same_sp else '!='} innovation {'==' if same_key else '!='}", flush=True)
    if not (same_pop and same_sp and same_key):
        print("MISMATCH")
        sys.exit(1)
print(f"{G} generations bit-exact at pop {P}, N{N}/C{C}; device (evaluate + fitness read + step per "
      f"generation, host-synchronised) {t_dev:.1f} s, restatement {t_orc:.1f} s")
