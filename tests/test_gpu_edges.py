"""Edge cases of the host layer the reference's own tests touch: empty
populations, zero representatives, batch 1, genomes without (enabled)
connections, the widest node limit (N_max = 255, k_transform<8>)."""
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


def test_empty_population_and_zero_representatives(fnb):
    prob = ol.Problem(16, 40, [0, 1, 2], [3])
    schema = ol.SchemaSpec(["tanh"], ["sum"])
    eng = _engine(fnb, prob, schema)
    n0, c0 = prob.empty_pop(0)
    order, cnt = eng.transform(n0, c0)
    assert order.shape == (0, 16) and cnt.shape == (0,)
    X = np.zeros((5, 3))
    assert eng.batch_forward(n0, c0, X).values.shape == (0, 5, 1)
    assert eng.evaluate(n0, c0, X, np.zeros((5, 1)), fnb.FIT_NEG_MSE).shape == (0,)
    n, c = ol.random_genomes(3, schema, 6, 16, 40)
    d = eng.distance(n, c, n[:0], c[:0])
    assert d.shape == (6, 0)
    gn, gc, nk = eng.mutate(n0, c0, np.zeros((0, 4), dtype=np.uint32), fnb.MutationConfig(), 7)
    assert gn.shape == (0, 16, 5) and nk == 7


def test_genomes_without_enabled_connections_and_batch_one(fnb):
    """No enabled edge into an output: the reference aggregates the identity
    (sum 0, product 1, max 0 by the forward's fallback, mean 0) and applies
    act(resp * agg + bias) (network.hpp:256-262)."""
    prob = ol.Problem(8, 8, [0, 1], [2])
    schema = ol.SchemaSpec(["tanh", "sigmoid", "identity"], ["sum", "product", "max", "mean"])
    P = 12
    n = np.full((P, 8, 5), np.nan)
    c = np.full((P, 8, 4), np.nan)
    rng = np.random.default_rng(4)
    for p in range(P):
        n[p, 0] = [0, 0.0, 1.0, 0, 0]
        n[p, 1] = [1, 0.0, 1.0, 0, 0]
        n[p, 2] = [2, rng.normal(), rng.uniform(0.5, 2), p % 4, p % 3]
        if p % 2:  # a disabled connection only
            c[p, 0] = [0, 2, 0.0, rng.normal()]
    X = rng.uniform(-1, 1, size=(1, 2))
    want = ol.ref_batch_forward(prob, schema, n, c, X)[3] if ol.ref_available() else None
    got = _engine(fnb, prob, schema).batch_forward(n, c, X).values
    if want is not None:
        np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-5)
    assert got.shape == (P, 1, 1) and np.all(np.isfinite(got))


def test_widest_node_limit(fnb):
    """N_max = 255 (the ABI's limit: node rows are addressed by a byte):
    k_transform<8>, order and outputs against the reference."""
    prob = ol.Problem(255, 1024, [0, 1, 2], [3])
    schema = ol.RICH
    n, c = ol.random_genomes(255, schema, 24, 255, 1024, spec=(3, 1, 180, 0.03, 0.15))
    eng = _engine(fnb, prob, schema)
    order, cnt = eng.transform(n, c)
    X = np.random.default_rng(2).uniform(-1, 1, size=(40, 3))
    got = eng.batch_forward(n, c, X).values
    for i in range(24):
        r = ol.ref_transform(prob, schema, n[i], c[i]) if ol.ref_available() else \
            ol.oracle_transform(prob, schema, n[i], c[i])
        assert r["status"] == 0 and cnt[i] == r["order_count"]
        np.testing.assert_array_equal(order[i], r["order"])
    if ol.ref_available():
        st, bad, msg, want = ol.ref_batch_forward(prob, schema, n, c, X)
        assert st == 0, msg
        np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-5)
