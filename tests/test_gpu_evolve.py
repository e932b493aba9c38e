"""The device generation loop vs the frozen CPU restatement (oracle/evolution.c).

SPEC-only stages have no reference code ("parity unpinned"),
so the bar is bit-exact equality with the restatement, which itself is built
on oracle functions pinned to the reference.  Both sides receive the SAME
fitness vector each generation: the device evaluates it, the
CPU loop is handed a copy.  Checked every generation: the whole population
(node and connection tensors, bit for bit), species ids / spawn counts /
best fitness / stagnation counters, and the innovation counter.
"""
import numpy as np
import pytest

import oracle_lib as ol

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fnb():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2504_08339_b200 as m
    return m


def _mut(fnb, kw):
    m = fnb.MutationConfig()
    for k, v in kw.items():
        setattr(m, k, fnb.AttrMutation(*v) if isinstance(v, tuple) else v)
    return m


CASES = [
    # (name, pop, limits, threshold, max_species, max_stagnation, mutation overrides, generations)
    ("default", 200, (24, 80), 3.5, 10, 15, {}, 12),
    ("many-species", 240, (24, 80), 0.6, 10, 15, dict(node_add=0.5, conn_add=0.6), 12),
    ("stagnation", 160, (20, 60), 0.8, 6, 1, dict(node_delete=0.2, conn_delete=0.2), 12),
    ("overflow", 120, (20, 60), 0.05, 4, 3, dict(activation_replace_rate=0.2), 10),
]


@pytest.mark.parametrize("name,P,limits,th,ms,stag,mkw,G", CASES)
def test_generation_loop_bit_exact(fnb, name, P, limits, th, ms, stag, mkw, G):
    from paper_2504_08339_b200.evolve import Evolver, NeatConfig
    from paper_2504_08339_b200.synthetic import regression_dataset
    schema_acts = ["tanh", "sigmoid", "identity"]
    prob = ol.Problem(limits[0], limits[1], [0, 1, 2], [3])
    schema = ol.SchemaSpec(schema_acts, ["sum", "product"])
    eng = fnb.Engine(fnb.GenomeLimits(*limits), [0, 1, 2], [3], fnb.AttributeSchema(schema_acts, ["sum", "product"]))
    cfg = NeatConfig(pop_size=P, max_species=ms, compatibility_threshold=th, max_stagnation=stag,
                     mutation=_mut(fnb, mkw), output_activation=1)
    ev = Evolver(eng, cfg, seed=2024)
    ocfg = ol.neat_cfg(P, max_species=ms, threshold=th, max_stagnation=stag, output_activation=1,
                       mutation=ol.mut_cfg(**mkw))
    orc = ol.OracleEvolution(prob, schema, ocfg, seed=2024)
    ev.init_population()
    orc.init_population()
    gn, gc = ev.population()
    np.testing.assert_array_equal(gn, orc.nodes)
    np.testing.assert_array_equal(gc, orc.conns)
    X, Y = regression_dataset(64, 3, 1, seed=5)
    for g in range(G):
        ev.evaluate(X, Y)
        fit = ev.fitness()
        orc.step(fit)
        ev.step()
        gn, gc = ev.population()
        np.testing.assert_array_equal(gn, orc.nodes, err_msg=f"{name} gen {g} nodes")
        np.testing.assert_array_equal(gc, orc.conns, err_msg=f"{name} gen {g} conns")
        sp, so = ev.species(), orc.species_view()
        assert sp["count"] == so["count"], (name, g)
        np.testing.assert_array_equal(sp["ids"], so["ids"])
        np.testing.assert_array_equal(sp["spawn"], so["spawn"])
        np.testing.assert_array_equal(sp["best"], so["best"])
        np.testing.assert_array_equal(sp["stagnation"], so["stagnation"])
        assert ev.state()[1] == orc.innov.next_key, (name, g)
        assert int(np.sum(sp["spawn"])) == P


def test_xor_evolves(fnb):
    """SPEC.md:441-449 shape: XOR with a bias input; fitness 4 - SSE rises."""
    from paper_2504_08339_b200.evolve import NeatConfig, evolve
    from paper_2504_08339_b200.synthetic import xor_dataset
    eng = fnb.Engine(fnb.GenomeLimits(16, 32), [0, 1, 2], [3], fnb.AttributeSchema(["sigmoid", "tanh"], ["sum"]))
    X, Y = xor_dataset(bias_input=True)
    cfg = NeatConfig(pop_size=1000, generation_limit=60, fitness_target=3.9)
    best, fit, stats = evolve(eng, cfg, seed=0, X=X, Y=Y, kind=fnb.FIT_OFFSET_SSE, offset=4.0)
    assert stats[-1].best >= stats[0].best
    assert fit > 3.0


def test_c1_xor_100_generations_bit_exact(fnb):
    """North-star bar on BASELINE config 1 (XOR, pop 1000, N_max=16, C_max=32,
    100 generations): the device evolution state equals the frozen CPU
    restatement bit for bit after EVERY generation -- population tensors,
    species table and innovation counter -- with the device's fitness
    (4 - SSE) handed to both sides."""
    from paper_2504_08339_b200.evolve import Evolver, NeatConfig
    from paper_2504_08339_b200.synthetic import xor_dataset
    acts, aggs = ["sigmoid", "tanh"], ["sum"]
    prob = ol.Problem(16, 32, [0, 1, 2], [3])
    schema = ol.SchemaSpec(acts, aggs)
    eng = fnb.Engine(fnb.GenomeLimits(16, 32), [0, 1, 2], [3], fnb.AttributeSchema(acts, aggs))
    P = 1000
    # threshold 1.0 (paper default 3.5 keeps XOR-sized genomes in one species)
    ev = Evolver(eng, NeatConfig(pop_size=P, compatibility_threshold=1.0), seed=11)
    orc = ol.OracleEvolution(prob, schema, ol.neat_cfg(P, threshold=1.0), seed=11)
    ev.init_population()
    orc.init_population()
    X, Y = xor_dataset(bias_input=True)
    species_seen = set()
    for g in range(100):
        ev.evaluate(X, Y, fnb.FIT_OFFSET_SSE, 4.0)
        fit = ev.fitness()
        orc.step(fit)
        ev.step()
        gn, gc = ev.population()
        # bit for bit, NaN padding included
        assert np.array_equal(gn.view(np.uint64), orc.nodes.view(np.uint64)), f"gen {g} nodes"
        assert np.array_equal(gc.view(np.uint64), orc.conns.view(np.uint64)), f"gen {g} conns"
        sp, so = ev.species(), orc.species_view()
        assert sp["count"] == so["count"] and np.array_equal(sp["ids"], so["ids"]), g
        assert np.array_equal(sp["spawn"], so["spawn"]) and np.array_equal(sp["best"], so["best"]), g
        assert ev.state()[1] == orc.innov.next_key, g
        species_seen.add(int(sp["count"]))
    assert ev.state()[0] == 100
    assert max(species_seen) > 1  # the run exercised speciation, not a single species


@pytest.mark.parametrize("parts", [1, 2, 3])
def test_split_step_equals_step(fnb, parts):
    """fnb_evolver_step_front / step_back(lo, hi) / step_commit -- the sharded
    reproduction of distributed.py -- over `parts` slot ranges on one GPU give
    the population, species table and innovation counter of fnb_evolver_step
    bit for bit, generation after generation."""
    from paper_2504_08339_b200.distributed import shard_bounds
    from paper_2504_08339_b200.evolve import Evolver, NeatConfig
    from paper_2504_08339_b200.synthetic import regression_dataset
    acts = ["tanh", "sigmoid", "identity"]
    eng = fnb.Engine(fnb.GenomeLimits(24, 80), [0, 1, 2], [3], fnb.AttributeSchema(acts, ["sum", "product"]))
    m = fnb.MutationConfig()
    m.node_add, m.conn_add, m.node_delete = 0.5, 0.6, 0.1
    cfg = NeatConfig(pop_size=301, compatibility_threshold=0.8, max_species=8, mutation=m)
    a, b = Evolver(eng, cfg, seed=99), Evolver(eng, cfg, seed=99)
    a.init_population()
    b.init_population()
    X, Y = regression_dataset(64, 3, 1, seed=4)
    for g in range(8):
        a.evaluate(X, Y)
        b.set_fitness(a.fitness())
        a.step()
        b.step_front()
        for r in range(parts):
            b.step_back(*shard_bounds(301, parts, r))
        b.step_commit()
        an, ac = a.population()
        bn, bc = b.population()
        assert np.array_equal(an.view(np.uint64), bn.view(np.uint64)), g
        assert np.array_equal(ac.view(np.uint64), bc.view(np.uint64)), g
        sa, sb = a.species(), b.species()
        assert sa["count"] == sb["count"] and np.array_equal(sa["spawn"], sb["spawn"]), g
        assert a.state() == b.state(), g
    # the next-population views alias the library's buffer
    n_view, c_view = b.next_population_d()
    assert tuple(n_view.shape) == (301, 24, 5) and tuple(c_view.shape) == (301, 80, 4)


@pytest.mark.parametrize("name,P,limits,inputs,th,G", [
    # P > 16,384: both stable sorts of the step take the CUB radix path (evolve.cu kCountRankMax)
    ("cub-sorts-P20000", 20000, (16, 32), 3, 0.6, 6),
    # BASELINE config 2 genome shape (N_max=64, C_max=256, 4 inputs)
    ("c2-shape-P2000", 2000, (64, 256), 4, 1.0, 10),
])
def test_generation_loop_bit_exact_large(fnb, name, P, limits, inputs, th, G):
    """The device loop against oracle/evolution.c at the populations and
    genome shapes the benchmarks run: whole population bit for bit (NaN
    padding included), species table and innovation counter, every generation."""
    from paper_2504_08339_b200.evolve import Evolver, NeatConfig
    from paper_2504_08339_b200.synthetic import regression_dataset
    acts, aggs = ["tanh", "sigmoid", "identity"], ["sum", "product"]
    ik = list(range(inputs))
    prob = ol.Problem(limits[0], limits[1], ik, [inputs])
    schema = ol.SchemaSpec(acts, aggs)
    eng = fnb.Engine(fnb.GenomeLimits(*limits), ik, [inputs], fnb.AttributeSchema(acts, aggs))
    mkw = dict(node_add=0.5, conn_add=0.6, node_delete=0.05, conn_delete=0.05)
    cfg = NeatConfig(pop_size=P, max_species=10, compatibility_threshold=th, mutation=_mut(fnb, mkw),
                     output_activation=1)
    ev = Evolver(eng, cfg, seed=77)
    orc = ol.OracleEvolution(prob, schema, ol.neat_cfg(P, max_species=10, threshold=th, output_activation=1,
                                                       mutation=ol.mut_cfg(**mkw)), seed=77)
    ev.init_population()
    orc.init_population()
    X, Y = regression_dataset(128, inputs, 1, seed=6)
    counts = set()
    for g in range(G):
        ev.evaluate(X, Y)
        fit = ev.fitness()
        orc.step(fit)
        ev.step()
        gn, gc = ev.population()
        assert np.array_equal(gn.view(np.uint64), orc.nodes.view(np.uint64)), f"{name} gen {g} nodes"
        assert np.array_equal(gc.view(np.uint64), orc.conns.view(np.uint64)), f"{name} gen {g} conns"
        sp, so = ev.species(), orc.species_view()
        assert sp["count"] == so["count"] and np.array_equal(sp["ids"], so["ids"]), (name, g)
        np.testing.assert_array_equal(sp["spawn"], so["spawn"])
        np.testing.assert_array_equal(sp["best"], so["best"])
        np.testing.assert_array_equal(sp["stagnation"], so["stagnation"])
        assert ev.state()[1] == orc.innov.next_key, (name, g)
        counts.add(int(sp["count"]))
    assert max(counts) > 1, f"{name}: the run never left one species"
