"""Device side of the multi-GPU loop (paper_2504_08339_b200/distributed.py).

* fitness is partition-invariant: evaluating genome ranges separately gives
  the same FP64 bits as evaluating the whole population (so N ranks
  reproduce the 1-GPU run);
* fnb_evolver_checksum matches its host restatement;
* ShardedGeneration + DeviceShardBackend at world size 1 steps exactly like
  the plain Evolver loop.
"""
import numpy as np
import pytest

from test_distributed import host_checksum

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2504_08339_b200 as fnb
    from paper_2504_08339_b200.evolve import Evolver, NeatConfig
    return torch, fnb, Evolver, NeatConfig


def _evolver(env, P, seed=5):
    torch, fnb, Evolver, NeatConfig = env
    eng = fnb.Engine(fnb.GenomeLimits(24, 80), [0, 1, 2], [3], fnb.AttributeSchema(["tanh", "sigmoid"], ["sum"]))
    m = fnb.MutationConfig()
    m.node_add, m.conn_add = 0.5, 0.7
    ev = Evolver(eng, NeatConfig(pop_size=P, compatibility_threshold=1.0, mutation=m, output_activation=1), seed)
    ev.init_population()
    return eng, ev


@pytest.mark.parametrize("B", [5, 32, 100, 1024])
def test_fitness_partition_invariant(env, B):
    torch = env[0]
    from paper_2504_08339_b200.synthetic import regression_dataset
    P = 600
    eng, ev = _evolver(env, P)
    for _ in range(3):  # grow some structure
        ev.set_fitness(np.random.default_rng(1).normal(size=P))
        ev.step()
    X, Y = regression_dataset(B, 3, 1, seed=9)
    Xd = torch.tensor(X, dtype=torch.float32, device="cuda")
    Yd = torch.tensor(Y, dtype=torch.float32, device="cuda")
    ev.evaluate_d(Xd, Yd)
    whole = ev.fitness()
    parts = []
    for lo, hi in [(0, 1), (1, 77), (77, 300), (300, P)]:
        out = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
        ev.evaluate_range_d(lo, hi, Xd, Yd, out)
        torch.cuda.synchronize()
        parts.append(out.cpu().numpy())
    np.testing.assert_array_equal(np.concatenate(parts), whole)


def test_checksum_matches_host(env):
    eng, ev = _evolver(env, 200)
    ev.set_fitness(np.linspace(-1, 0, 200))
    ev.step()
    n, c = ev.population()
    gen, nk = ev.state()
    want = host_checksum(n, c) ^ ((nk & 0xFFFFFFFF) << 32) ^ (gen & 0xFFFFFFFF)
    assert ev.checksum() == want


def test_sharded_world1_matches_plain_loop(env):
    torch = env[0]
    from paper_2504_08339_b200.distributed import DeviceShardBackend, ShardedGeneration
    from paper_2504_08339_b200.synthetic import regression_dataset
    P, G = 300, 5
    X, Y = regression_dataset(64, 3, 1, seed=4)
    Xd = torch.tensor(X, dtype=torch.float32, device="cuda")
    Yd = torch.tensor(Y, dtype=torch.float32, device="cuda")
    _, a = _evolver(env, P, seed=8)
    _, b = _evolver(env, P, seed=8)
    sg = ShardedGeneration(DeviceShardBackend(b, Xd, Yd))
    for _ in range(G):
        a.evaluate_d(Xd, Yd)
        fa = a.fitness()
        a.step()
        fb = sg.generation().cpu().numpy()
        np.testing.assert_array_equal(fa, fb)
    assert a.checksum() == b.checksum()
    assert sg.replicas_agree()
