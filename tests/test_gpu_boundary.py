"""Boundary behaviour through the C ABI on the GPU: the caller's
InnovationTable (ops.hpp:145-175), invalid genomes in reused buffers, the
evolver's evaluation errors (network.hpp:122-268, "errors
abort with context"), and the empty dataset."""
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


def _engine(fnb, prob, schema):
    return fnb.Engine(fnb.GenomeLimits(prob.max_nodes, prob.max_conns), prob.input_keys, prob.output_keys,
                      fnb.AttributeSchema(list(schema.activations), list(schema.aggregations)))


def test_mutate_with_table_matches_reference(fnb):
    """fnb_mutate_table with a fresh InnovationTable == the reference's slot-order loop."""
    schema = ol.SchemaSpec(["tanh", "sigmoid", "identity"], ["sum", "product"])
    prob = ol.Problem(24, 80, [0, 1, 2], [3])
    nodes, conns = ol.random_genomes(99, schema, 128, 24, 80)
    keys = np.stack([ol.key_words(ol.key_split(ol.key_seed(5), p)) for p in range(128)])
    kw = dict(node_add=0.7, conn_add=0.5, node_delete=0.1)
    st, bad, nk_ref, wn, wc = ol.mutate_population(prob, schema, nodes, conns, keys, ol.mut_cfg(**kw), 500,
                                                   use_ref=ol.ref_available())
    assert st == 0
    m = fnb.MutationConfig()
    for k, v in kw.items():
        setattr(m, k, v)
    table = fnb.InnovationTable(500)
    gn, gc, nk = _engine(fnb, prob, schema).mutate(nodes, conns, keys, m, table=table)
    assert nk == nk_ref == table.next_key()
    np.testing.assert_array_equal(gn, wn)
    np.testing.assert_array_equal(gc, wc)
    # one memo entry per distinct split pair, keys handed out consecutively
    assert sorted(table._assignments.values()) == list(range(500, nk))


def test_mutate_table_memo_is_used(fnb):
    """A pair already in the caller's table keeps its key (ops.hpp:149-153):
    pre-assign every pair a fresh run would split, under other keys."""
    schema = ol.SchemaSpec(["tanh"], ["sum"])
    prob = ol.Problem(20, 60, [0, 1], [2])
    nodes, conns = ol.random_genomes(12, schema, 64, 20, 60)
    keys = np.stack([ol.key_words(ol.key_split(ol.key_seed(8), p)) for p in range(64)])
    m = fnb.MutationConfig()
    m.node_add = 1.0
    eng = _engine(fnb, prob, schema)
    fresh = fnb.InnovationTable(1000)
    a_n, a_c, _ = eng.mutate(nodes, conns, keys, m, table=fresh)
    seeded = fnb.InnovationTable(3000)
    remap = {}
    for pair, k in sorted(fresh._assignments.items(), key=lambda t: -t[1]):  # reversed order -> other keys
        remap[k] = seeded.get_or_assign(*pair)
    before = seeded.next_key()
    b_n, b_c, nk = eng.mutate(nodes, conns, keys, m, table=seeded)
    assert nk == before  # no new key handed out
    # identical genomes up to the key renaming
    f = np.vectorize(lambda x: remap.get(int(x), x) if not np.isnan(x) else x)
    np.testing.assert_array_equal(f(a_n[..., 0]), b_n[..., 0])
    np.testing.assert_array_equal(f(a_c[..., :2]), b_c[..., :2])
    np.testing.assert_array_equal(a_n[..., 1:], b_n[..., 1:])
    np.testing.assert_array_equal(a_c[..., 2:], b_c[..., 2:])


def test_invalid_genomes_after_valid_population_same_buffers(fnb):
    """Transform failures leave no stale value-slot count behind:
    the same engine evaluates a valid population, then one with cycles and
    dangling endpoints interleaved, then the valid one again -- valid genomes'
    fitness is unchanged bit for bit and the failing genome is reported."""
    import torch
    from test_oracle_vs_ref import _corrupt
    from paper_2504_08339_b200.synthetic import regression_dataset
    prob = ol.Problem(64, 256, [0, 1, 2, 3], [4])
    schema = ol.SchemaSpec(["tanh"], ["sum"])
    from paper_2504_08339_b200.synthetic import synthetic_population
    nodes, conns = synthetic_population(600, 64, 256, fill=0.9, seed=31)
    X, Y = regression_dataset(256, seed=2)
    eng = _engine(fnb, prob, schema)
    f0 = eng.evaluate(nodes, conns, X, Y, fnb.FIT_NEG_MSE)
    rng = np.random.default_rng(3)
    bn, bc = nodes.copy(), conns.copy()
    bad_rows = list(range(1, 600, 7))
    for i in bad_rows:
        bn[i], bc[i] = _corrupt(nodes[i], conns[i], rng, "cycle" if i % 2 else "dangling")
    with pytest.raises(fnb.FlatneatError) as ei:
        eng.evaluate(bn, bc, X, Y, fnb.FIT_NEG_MSE)
    assert ei.value.index == 1 and ei.value.code in ("cycle_detected", "dangling_endpoint")
    # device layer on the mixed population: the valid genomes' fitness is untouched
    dev = torch.device("cuda", 0)
    tn = torch.as_tensor(bn, device=dev)
    tc = torch.as_tensor(bc, device=dev)
    nets = eng.alloc_nets(600)
    eng.transform_d(tn, tc, nets)
    fit = torch.full((600,), float("nan"), dtype=torch.float64, device=dev)
    Xf = torch.as_tensor(X, dtype=torch.float32, device=dev)
    Yf = torch.as_tensor(Y, dtype=torch.float32, device=dev)
    eng.forward_d(nets, 600, Xf, Yf, fnb.FIT_NEG_MSE, fitness=fit)
    torch.cuda.synchronize()
    got = fit.cpu().numpy()
    ok = np.setdiff1d(np.arange(600), bad_rows)
    np.testing.assert_array_equal(got[ok], f0[ok])
    f1 = eng.evaluate(nodes, conns, X, Y, fnb.FIT_NEG_MSE)
    np.testing.assert_array_equal(f1, f0)


def test_evolver_evaluate_reports_errors(fnb):
    """fnb_evolver_evaluate: transform errors with the genome index, then
    non-finite inputs, then the empty dataset."""
    from test_oracle_vs_ref import _corrupt
    from paper_2504_08339_b200.evolve import Evolver, NeatConfig
    prob = ol.Problem(20, 60, [0, 1, 2], [3])
    schema = ol.SchemaSpec(["tanh", "identity"], ["sum"])
    nodes, conns = ol.random_genomes(44, schema, 50, 20, 60)
    eng = _engine(fnb, prob, schema)
    ev = Evolver(eng, NeatConfig(pop_size=50), seed=1)
    rng = np.random.default_rng(4)
    n2, c2 = nodes.copy(), conns.copy()
    n2[17], c2[17] = _corrupt(nodes[17], conns[17], rng, "cycle")
    r = ol.ref_transform(prob, schema, n2[17], c2[17]) if ol.ref_available() else \
        ol.oracle_transform(prob, schema, n2[17], c2[17])
    ev.set_population(n2, c2)
    X = rng.uniform(-1, 1, size=(32, 3))
    Y = rng.uniform(-1, 1, size=(32, 1))
    with pytest.raises(fnb.FlatneatError) as ei:
        ev.evaluate(X, Y)
    assert ei.value.index == 17 and ei.value.code == "cycle_detected" and str(ei.value) == r["msg"]
    ev.set_population(nodes, conns)
    Xn = X.copy()
    Xn[3, 1] = np.nan
    with pytest.raises(fnb.FlatneatError) as ei:
        ev.evaluate(Xn, Y)
    assert ei.value.code == "non_finite_input"
    with pytest.raises(fnb.FlatneatError) as ei:
        ev.evaluate(X[:0], Y[:0])
    assert ei.value.code == "empty_dataset"
    ev.evaluate(X, Y)  # and a clean evaluation afterwards
    assert np.all(np.isfinite(ev.fitness()))
    # the device-input variant reports through eval_check
    import torch
    Xd = torch.as_tensor(Xn, dtype=torch.float32, device="cuda")
    Yd = torch.as_tensor(Y, dtype=torch.float32, device="cuda")
    ev.evaluate_d(Xd, Yd)
    with pytest.raises(fnb.FlatneatError) as ei:
        ev.eval_check()
    assert ei.value.code == "non_finite_input"


def test_evaluate_empty_dataset(fnb):
    prob = ol.Problem(16, 32, [0, 1], [2])
    schema = ol.SchemaSpec(["tanh"], ["sum"])
    nodes, conns = ol.random_genomes(1, schema, 4, 16, 32)
    with pytest.raises(fnb.FlatneatError) as ei:
        _engine(fnb, prob, schema).evaluate(nodes, conns, np.zeros((0, 2)), np.zeros((0, 1)), fnb.FIT_NEG_MSE)
    assert ei.value.code == "empty_dataset"
