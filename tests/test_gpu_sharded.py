"""The generation step sharded over ranks (distributed.ShardedEvolution,
fnb_evolver_shard_*): each rank owns a genome block, and only fitness,
species statistics, founders, new representatives and the selected parents
cross between ranks.  Bar: the one-process device step, bit for bit --
population shards, species table, innovation counter -- at world size 1 and
at world size 2 (two processes on one GPU over gloo: the same collectives
NCCL runs on a multi-GPU box)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ACTS, AGGS = ["tanh", "sigmoid", "identity"], ["sum", "product"]
CASES = {
    # name: (P, limits, threshold, max_species, max_stagnation, generations)
    "founding": (301, (24, 80), 0.7, 8, 15, 8),
    "stagnation": (240, (20, 60), 0.9, 6, 1, 8),
    "overflow": (150, (20, 60), 0.05, 4, 3, 6),
    # BASELINE config 2 genome shape, 2,000 genomes: many founding rounds across both shards
    "c2-shape": (2000, (64, 256), 1.2, 10, 15, 4),
}


def _make(case, seed=31):
    import paper_2504_08339_b200 as fnb
    from paper_2504_08339_b200.evolve import Evolver, NeatConfig
    P, limits, th, ms, stag, G = CASES[case]
    ni = 4 if limits[0] >= 64 else 3
    eng = fnb.Engine(fnb.GenomeLimits(*limits), list(range(ni)), [ni], fnb.AttributeSchema(ACTS, AGGS))
    m = fnb.MutationConfig()
    m.node_add, m.conn_add, m.node_delete, m.conn_delete = 0.4, 0.6, 0.05, 0.05
    cfg = NeatConfig(pop_size=P, compatibility_threshold=th, max_species=ms, max_stagnation=stag, mutation=m)
    ev = Evolver(eng, cfg, seed=seed)
    ev.init_population()
    return eng, ev, G


def _data(ni=3):
    import torch
    from paper_2504_08339_b200.synthetic import regression_dataset
    X, Y = regression_dataset(64, ni, 1, seed=9)
    return (torch.as_tensor(X, dtype=torch.float32, device="cuda"),
            torch.as_tensor(Y, dtype=torch.float32, device="cuda"))


def _reference_run(case):
    """The one-process device loop: evaluate + fnb_evolver_step per generation."""
    eng, ev, G = _make(case)
    X, Y = _data(eng.num_inputs)
    out = []
    for _ in range(G):
        ev.evaluate_d(X, Y)
        ev.step()
        n, c = ev.population()
        sp = ev.species()
        out.append((n, c, sp["ids"].copy(), sp["spawn"].copy(), sp["best"].copy(), ev.state()))
    return out


def _sharded_run(case, world=1, rank=0):
    from paper_2504_08339_b200.distributed import ShardedEvolution
    eng, ev, G = _make(case)
    X, Y = _data(eng.num_inputs)
    se = ShardedEvolution(ev, X, Y)
    out = []
    for _ in range(G):
        se.generation()
        n, c = ev.population()
        sp = ev.species()
        out.append((n[se.lo:se.hi], c[se.lo:se.hi], sp["ids"].copy(), sp["spawn"].copy(), sp["best"].copy(),
                    ev.state(), se.lo, se.hi))
    return out


def _check(ref, got, lo_hi=None):
    for g, (r, s) in enumerate(zip(ref, got)):
        lo, hi = s[6], s[7]
        assert np.array_equal(r[0][lo:hi].view(np.uint64), s[0].view(np.uint64)), f"gen {g} nodes"
        assert np.array_equal(r[1][lo:hi].view(np.uint64), s[1].view(np.uint64)), f"gen {g} conns"
        for k in (2, 3, 4):
            assert np.array_equal(r[k], s[k]), (g, k)
        assert r[5] == s[5], g


@pytest.fixture(scope="module")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("case", sorted(CASES))
def test_sharded_world1_equals_step(cuda, case):
    _check(_reference_run(case), _sharded_run(case))


def _worker(rank, world, port, case, q):
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        q.put((rank, _sharded_run(case, world, rank)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", sorted(CASES))
def test_sharded_world2_equals_one_process(cuda, case):
    import torch.multiprocessing as mp
    ref = _reference_run(case)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        _check(ref, res[r])
    assert res[0][-1][7] == res[1][-1][6]  # the shards tile the population
