"""BASELINE config 5 at full size (pop 100k, N_max=128, C_max=1024) on the
device: properties that do not need a CPU oracle at that size (the oracle
runs the same shapes on 4,000 genomes, scripts/validate_c5_shape.py):
the three ways of running a generation -- fnb_evolve's CUDA graphs, the
evaluate / step calls, the sharded step at world size 1 -- give the same
population bit for bit (checksums), every genome stays valid
(explain_invalid over all 100k), species sizes and spawn counts sum to the
population."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

P5, N5, C5 = 100_000, 128, 1024


@pytest.fixture(scope="module")
def setup():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2504_08339_b200 as fnb
    from paper_2504_08339_b200.synthetic import regression_dataset, synthetic_population
    n_h, c_h = synthetic_population(2_000, N5, C5, 0.75, 4, 1, seed=5)
    nodes = torch.from_numpy(n_h).cuda().repeat(P5 // 2_000, 1, 1)
    conns = torch.from_numpy(c_h).cuda().repeat(P5 // 2_000, 1, 1)
    X_h, Y_h = regression_dataset(256, 4, 1, seed=0)
    eng = fnb.Engine(fnb.GenomeLimits(N5, C5), [0, 1, 2, 3], [4], fnb.AttributeSchema())
    return fnb, eng, nodes, conns, X_h, Y_h


def _evolver(setup, seed=5):
    from paper_2504_08339_b200.evolve import Evolver, NeatConfig
    fnb, eng, nodes, conns, X_h, Y_h = setup
    ev = Evolver(eng, NeatConfig(pop_size=P5, compatibility_threshold=1.9), seed=seed)
    ev.set_population_d(nodes, conns)
    return ev


def test_c5_three_paths_agree_and_stay_valid(setup):
    import torch
    from paper_2504_08339_b200.distributed import ShardedEvolution
    fnb, eng, nodes, conns, X_h, Y_h = setup
    G = 2
    a = _evolver(setup)
    _, _, stats = a.run(X_h, Y_h, generation_limit=G)
    assert a.run_mode() == 2 and len(stats) == G
    ha = a.checksum()
    sp = a.species()
    assert int(np.sum(sp["sizes"])) == P5 and int(np.sum(sp["spawn"])) == P5
    assert a.validate() == -1
    a.close()
    b = _evolver(setup)
    Xd = torch.as_tensor(X_h, dtype=torch.float32, device="cuda")
    Yd = torch.as_tensor(Y_h, dtype=torch.float32, device="cuda")
    for _ in range(G):
        b.evaluate_d(Xd, Yd)
        b.eval_check()
        b.step()
    assert b.checksum() == ha
    b.close()
    c = _evolver(setup)
    se = ShardedEvolution(c, Xd, Yd)
    for _ in range(G):
        se.generation()
    assert c.checksum() == ha
    c.close()
