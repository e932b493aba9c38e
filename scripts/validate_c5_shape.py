"""BASELINE config 5 genome shapes (N_max=128, C_max=1024, fill 0.75): the
device generation loop against the frozen restatement oracle/evolution.c,
both sides given the device's fitness each generation.  The restatement's
single-threaded distance / crossover / mutate cannot run pop 100k in bounded
time, so the population is FNB_VALIDATE_P genomes (default 4,000); the
kernels run the same C5-shape code paths (k_transform<4>, the N128 forward
geometry, K3 at C_max=1024, K5 / K6 with 1-2-warp CTAs).  Population,
species table and innovation counter are compared bit for bit every
generation.

    python scripts/validate_c5_shape.py [generations] > profiles/r02_validate_c5_shape.txt
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

G = int(sys.argv[1]) if len(sys.argv) > 1 else 3
P, N, C, B = int(os.environ.get("FNB_VALIDATE_P", "4000")), 128, 1024, 1024
acts, aggs = ["tanh"], ["sum"]
eng = fnb.Engine(fnb.GenomeLimits(N, C), [0, 1, 2, 3], [4], fnb.AttributeSchema(acts, aggs))
TH = float(os.environ.get("FNB_VALIDATE_TH", "1.9"))  # random C5 topologies sit ~2.0 apart: several species
ev = Evolver(eng, NeatConfig(pop_size=P, compatibility_threshold=TH), seed=2025)
orc = ol.OracleEvolution(ol.Problem(N, C, [0, 1, 2, 3], [4]), ol.SchemaSpec(acts, aggs), ol.neat_cfg(P, threshold=TH), seed=2025)
from paper_2504_08339_b200.synthetic import synthetic_population  # noqa: E402
n0, c0 = synthetic_population(P, N, C, 0.75, 4, 1, n_act=1, n_agg=1, seed=55)
ev.set_population(n0, c0)
orc.set_population(n0, c0)
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
