"""SPEC evolve on the device -- fnb_evolve, one CUDA graph
per generation with the termination test on the device -- and
checkpoint/resume (fnb_evolver_get_state / set_state + the checkpoint wire
document): 10 generations -> save -> restore -> 10 more equals 20
uninterrupted generations bit for bit."""
import os

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


ACTS, AGGS = ["tanh", "sigmoid", "identity"], ["sum", "product"]


def _setup(fnb, P=300, seed=21, **kw):
    from paper_2504_08339_b200.evolve import Evolver, NeatConfig
    from paper_2504_08339_b200.synthetic import regression_dataset
    eng = fnb.Engine(fnb.GenomeLimits(24, 80), [0, 1, 2], [3], fnb.AttributeSchema(ACTS, AGGS))
    m = fnb.MutationConfig()
    m.node_add, m.conn_add, m.node_delete, m.conn_delete = 0.4, 0.5, 0.05, 0.05
    cfg = NeatConfig(pop_size=P, compatibility_threshold=0.9, max_species=8, mutation=m, **kw)
    X, Y = regression_dataset(96, 3, 1, seed=3)
    return eng, cfg, Evolver(eng, cfg, seed=seed), X, Y


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def _stats_key(stats):
    return [(s.generation, s.best, s.mean, s.std, s.best_index, s.species_count, s.species_sizes) for s in stats]


@pytest.mark.parametrize("graph", ["1", "0"])
def test_run_equals_step_loop(fnb, graph, monkeypatch):
    """fnb_evolve (conditional-node generation graph, or with FNB_GEN_GRAPH=0
    the evaluate graph + host check + step graph) equals the evaluate / step
    loop through the C ABI bit for bit, RunStats included."""
    monkeypatch.setenv("FNB_GEN_GRAPH", graph)
    eng, cfg, a, X, Y = _setup(fnb)
    _, _, b, _, _ = _setup(fnb)
    a.init_population()
    b.init_population()
    _, _, stats = a.run(X, Y, generation_limit=8)
    assert a.run_mode() == (2 if graph == "1" else 1)
    assert [s.generation for s in stats] == list(range(8))
    for g in range(8):
        b.evaluate(X, Y)
        f = b.fitness()
        assert stats[g].best == f.max() and stats[g].best_index == int(np.argmax(f))
        assert abs(stats[g].mean - f.mean()) <= 1e-12 * abs(f.mean()) + 1e-15
        b.step()
        assert stats[g].species_count == b.species()["count"]
    an, ac = a.population()
    bn, bc = b.population()
    assert np.array_equal(_bits(an), _bits(bn)) and np.array_equal(_bits(ac), _bits(bc))
    assert a.state() == b.state() == (8, b.state()[1])


def test_checkpoint_resume_bit_exact(fnb):
    """10 generations -> save_checkpoint -> load into a NEW engine and evolver
    (another seed at creation: the checkpoint restores it) -> 10 more ==
    20 uninterrupted generations: population, species table, innovation
    counter, generation and the RunStats of generations 10-19."""
    eng, cfg, full, X, Y = _setup(fnb)
    full.init_population()
    _, _, s_full = full.run(X, Y, generation_limit=20)

    _, _, first, _, _ = _setup(fnb)
    first.init_population()
    first.run(X, Y, generation_limit=10)
    text = first.save_checkpoint()
    first.close()
    _, _, resumed, _, _ = _setup(fnb, seed=999)
    resumed.load_checkpoint(text)
    assert resumed.state()[0] == 10
    _, _, s_res = resumed.run(X, Y, generation_limit=10)

    assert _stats_key(s_res) == _stats_key(s_full[10:])
    fn, fc = full.population()
    rn, rc = resumed.population()
    assert np.array_equal(_bits(fn), _bits(rn)) and np.array_equal(_bits(fc), _bits(rc))
    sf, sr = full.get_state(), resumed.get_state()
    assert sf[0] == sr[0]
    assert np.array_equal(_bits(sf[1]), _bits(sr[1])) and np.array_equal(_bits(sf[2]), _bits(sr[2]))
    # the document itself round-trips byte for byte
    from paper_2504_08339_b200.wire import load_checkpoint, save_checkpoint
    st, a, b, n, c, meta = load_checkpoint(text)
    assert save_checkpoint(st, a, b, n, c, meta["input_keys"], meta["output_keys"], meta["activations"],
                           meta["aggregations"]) == text


def test_evolve_spec_examples(fnb):
    """fitness_target = +inf, generation_limit = 5 -> exactly
    5 generations of stats; a constant-fitness problem -> the best genome is
    the argmax with the lowest-index tie-break; same seed twice -> identical
    RunStats and identical best-genome serialization."""
    from paper_2504_08339_b200.evolve import evolve
    from paper_2504_08339_b200.wire import save_genome
    eng, cfg, _, X, Y = _setup(fnb)
    cfg.generation_limit = 5
    best, fit, stats = evolve(eng, cfg, seed=4, X=X, Y=Y)
    assert len(stats) == 5
    best2, fit2, stats2 = evolve(eng, cfg, seed=4, X=X, Y=Y)
    assert _stats_key(stats) == _stats_key(stats2) and fit == fit2
    assert save_genome(*best, [0, 1, 2], [3], ACTS, AGGS) == save_genome(*best2, [0, 1, 2], [3], ACTS, AGGS)
    seen = []
    best3, fit3, stats3 = evolve(eng, cfg, seed=4, fitness_fn=lambda n, c: (seen.append(n[0].copy()), np.zeros(len(n)))[1])
    assert len(stats3) == 5 and fit3 == 0.0 and all(s.best_index == 0 for s in stats3)
    assert np.array_equal(_bits(best3[0]), _bits(seen[-1]))


def test_evolve_stops_before_reproducing(fnb):
    """Termination checks fitness BEFORE reproduction: a target
    every genome meets stops after one evaluation, with no step taken."""
    eng, cfg, ev, X, Y = _setup(fnb)
    ev.init_population()
    n0, c0 = ev.population()
    best, fit, stats = ev.run(X, Y, fitness_target=-1e300, generation_limit=50)
    assert len(stats) == 1 and ev.state()[0] == 0
    n1, c1 = ev.population()
    assert np.array_equal(_bits(n0), _bits(n1)) and np.array_equal(_bits(c0), _bits(c1))
    i = stats[0].best_index
    assert np.array_equal(_bits(best[0]), _bits(n0[i])) and np.array_equal(_bits(best[1]), _bits(c0[i]))


def test_evolve_error_context(fnb):
    """Evaluation errors abort with generation and genome context."""
    from test_oracle_vs_ref import _corrupt
    eng, cfg, ev, X, Y = _setup(fnb, P=60)
    schema = ol.SchemaSpec(ACTS, AGGS)
    n, c = ol.random_genomes(5, schema, 60, 24, 80)
    n[17], c[17] = _corrupt(n[17], c[17], np.random.default_rng(2), "cycle")
    ev.set_population(n, c)
    with pytest.raises(fnb.FlatneatError) as ei:
        ev.run(X, Y, generation_limit=3)
    assert ei.value.code == "cycle_detected" and ei.value.index == 17
    assert "generation 0, genome 17: cycle " in str(ei.value)


def test_run_graph_cache_follows_the_problem(fnb):
    """The generation graphs cached across fnb_evolve calls bake in the
    problem's device buffers: a run on another dataset (another batch size,
    so the input buffer moves) must equal the step loop on that dataset."""
    from paper_2504_08339_b200.synthetic import regression_dataset
    eng, cfg, a, X, Y = _setup(fnb, P=200)
    _, _, b, _, _ = _setup(fnb, P=200)
    a.init_population()
    b.init_population()
    a.run(X, Y, generation_limit=3)
    for _ in range(3):
        b.evaluate(X, Y)
        b.step()
    X2, Y2 = regression_dataset(300, 3, 1, seed=11)
    _, _, stats = a.run(X2, Y2, generation_limit=3)
    for g in range(3):
        b.evaluate(X2, Y2)
        f = b.fitness()
        assert stats[g].best == f.max()
        b.step()
    an, ac = a.population()
    bn, bc = b.population()
    assert np.array_equal(_bits(an), _bits(bn)) and np.array_equal(_bits(ac), _bits(bc))


def test_checkpoint_before_any_step(fnb):
    """A checkpoint of a fresh population (no species yet) restores and runs like the original."""
    eng, cfg, a, X, Y = _setup(fnb, P=150)
    a.init_population()
    text = a.save_checkpoint()
    _, _, b, _, _ = _setup(fnb, P=150, seed=7)
    b.load_checkpoint(text)
    _, _, sa = a.run(X, Y, generation_limit=4)
    _, _, sb = b.run(X, Y, generation_limit=4)
    assert _stats_key(sa) == _stats_key(sb)
    an, ac = a.population()
    bn, bc = b.population()
    assert np.array_equal(_bits(an), _bits(bn)) and np.array_equal(_bits(ac), _bits(bc))
