"""GPU parity for K6 (mutate) + K7 (innovation keys), bit-exact against the
reference's sequential slot-order mutate with one InnovationTable
(ops.hpp:169-175, 363-374) -- including every normal() draw, which needs
the glibc-exact log/cos of csrc/glibc_math.cuh."""
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


def _cfg(fnb, kw):
    m = fnb.MutationConfig()
    for k, v in kw.items():
        if isinstance(v, tuple):
            v = fnb.AttrMutation(*v)
        setattr(m, k, v)
    return m


CONFIGS = [
    {},
    dict(node_delete=0.15, conn_delete=0.15, activation_replace_rate=0.1, aggregation_replace_rate=0.1),
    dict(node_add=0.9, conn_add=0.9, node_delete=0.3, conn_delete=0.3),
    dict(node_add=0.0, conn_add=1.0, bias=(0.0, 1.0, 0.5, 0.0, 1.0), weight=(0.3, 2.0, 0.5, 0.5, 0.5)),
]


@pytest.mark.parametrize("cfgkw", CONFIGS)
# (20, 8200): C_max past 2^13, so K6 attrs keeps its normal list unpacked
@pytest.mark.parametrize("limits,seed", [((18, 60), 404), ((64, 256), 7), ((20, 8200), 3)])
def test_mutate_population_bit_exact(fnb, cfgkw, limits, seed):
    schema = ol.SchemaSpec(["tanh", "sigmoid", "identity"], ["sum", "product"])
    prob = ol.Problem(limits[0], limits[1], [0, 1, 2], [3])
    nodes, conns = ol.random_genomes(seed, schema, 160, *limits)
    eng = _engine(fnb, prob, schema)
    cfg_o = ol.mut_cfg(**cfgkw)
    cfg_g = _cfg(fnb, cfgkw)
    root = ol.key_seed(17)
    next_key = 1000
    use_ref = ol.ref_available()
    for step in range(3):
        keys = np.stack([ol.key_words(ol.key_split(ol.key_split(root, step), p)) for p in range(160)])
        st, bad, nk_ref, wn, wc = ol.mutate_population(prob, schema, nodes, conns, keys, cfg_o, next_key,
                                                       use_ref=use_ref)
        assert st == 0
        gn, gc, nk = eng.mutate(nodes, conns, keys, cfg_g, next_key)
        assert nk == nk_ref
        np.testing.assert_array_equal(gn, wn)
        np.testing.assert_array_equal(gc, wc)
        nodes, conns, next_key = gn, gc, nk


def test_mutate_duplicate_key_error_matches(fnb):
    """Restarting the innovation counter below existing keys -> duplicate_key
    at the same genome as the sequential reference (ops.hpp:21-22)."""
    schema = ol.SchemaSpec(["tanh"], ["sum"])
    prob = ol.Problem(20, 80, [0, 1, 2], [3])
    nodes, conns = ol.random_genomes(11, schema, 64, 20, 80)
    keys = np.stack([ol.key_words(ol.key_split(ol.key_seed(3), p)) for p in range(64)])
    cfg_o = ol.mut_cfg(node_add=1.0)
    st, bad, nk_ref, wn, wc = ol.mutate_population(prob, schema, nodes, conns, keys, cfg_o, 4,
                                                   use_ref=ol.ref_available())
    assert st == 1 + ol.ERRC.index("duplicate_key")
    with pytest.raises(fnb.FlatneatError) as ei:
        _engine(fnb, prob, schema).mutate(nodes, conns, keys, _cfg(fnb, dict(node_add=1.0)), 4)
    assert ei.value.code == "duplicate_key" and ei.value.index == bad
    gn, gc, nk = ei.value.partial
    assert nk == nk_ref
    np.testing.assert_array_equal(gn, wn)
    np.testing.assert_array_equal(gc, wc)


def test_mutation_known_answers(fnb):
    """test_ops.cpp:129-196: zero rates = identity; node split rule; saturated conn add."""
    schema = ol.SchemaSpec(["tanh", "identity"], ["sum"])
    prob = ol.Problem(6, 6, [0], [1])
    n = np.full((1, 6, 5), np.nan)
    n[0, 0] = [0, 0.0, 1.0, 0, 0]
    n[0, 1] = [1, 0.0, 1.0, 0, 0]
    c = np.full((1, 6, 4), np.nan)
    c[0, 0] = [0, 1, 1, 0.7]
    eng = _engine(fnb, prob, schema)
    split = _cfg(fnb, dict(node_add=1.0, conn_add=0.0, bias=(0, 0, 0, 0, 0), response=(1, 0, 0, 0, 0),
                           weight=(0, 1, 0.5, 0, 0)))
    gn, gc, nk = eng.mutate(n, c, ol.key_words(ol.key_seed(5))[None], split, 2)
    assert nk == 3
    rows = {(int(r[0]), int(r[1])): (r[2], r[3]) for r in gc[0] if not np.isnan(r[0])}
    assert rows == {(0, 1): (0.0, 0.7), (0, 2): (1.0, 1.0), (2, 1): (1.0, 0.7)}
    assert gn[0, 2, 0] == 2 and gn[0, 2, 1] == 0.0 and gn[0, 2, 2] == 1.0


@pytest.mark.parametrize("cfgkw", CONFIGS)
def test_mutate_c5_shape_bit_exact(fnb, cfgkw):
    """K6 + K7 at BASELINE config 5 shapes (N128/C1024, fill 0.75; K6 runs
    1-2-warp CTAs there): 3 slot-order steps x 4 mutation configs against
    the reference's mutate with one InnovationTable, every normal included."""
    from paper_2504_08339_b200.synthetic import synthetic_population
    schema = ol.SchemaSpec(["tanh", "sigmoid", "identity"], ["sum", "product"])
    prob = ol.Problem(128, 1024, [0, 1, 2, 3], [4])
    nodes, conns = synthetic_population(64, 128, 1024, fill=0.75, n_act=3, n_agg=2, seed=71)
    eng = _engine(fnb, prob, schema)
    cfg_o = ol.mut_cfg(**cfgkw)
    cfg_g = _cfg(fnb, cfgkw)
    root = ol.key_seed(72)
    next_key = 1000
    use_ref = ol.ref_available()
    for step in range(3):
        keys = np.stack([ol.key_words(ol.key_split(ol.key_split(root, step), p)) for p in range(64)])
        st, bad, nk_ref, wn, wc = ol.mutate_population(prob, schema, nodes, conns, keys, cfg_o, next_key,
                                                       use_ref=use_ref)
        assert st == 0
        gn, gc, nk = eng.mutate(nodes, conns, keys, cfg_g, next_key)
        assert nk == nk_ref
        np.testing.assert_array_equal(gn, wn)
        np.testing.assert_array_equal(gc, wc)
        nodes, conns, next_key = gn, gc, nk
