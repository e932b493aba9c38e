"""GPU parity for K1 (transform) and K2 (forward + fitness) through the C ABI.

Checker: the reference compiled from /root/reference (oracle/_ref) when
present, else the C restatement (oracle/liboracle.so) -- both pinned to each
other by tests/test_oracle_vs_ref.py.  Bars (north star): topological order,
error codes and messages bit-exact; outputs within rtol 1e-5 + atol 1e-5 of
the FP64 reference; fitness within rtol 1e-5.
"""
import os

import numpy as np
import pytest

import oracle_lib as ol

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-5, 1e-5


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


def _ref_transform(prob, schema, n, c):
    return ol.ref_transform(prob, schema, n, c) if ol.ref_available() else ol.oracle_transform(prob, schema, n, c)


def _ref_forward(prob, schema, n, c, X):
    if ol.ref_available():
        st, bad, msg, out = ol.ref_batch_forward(prob, schema, n, c, X)
        assert st == 0, msg
        return out
    outs = []
    for i in range(n.shape[0]):
        net = ol.oracle_transform(prob, schema, n[i], c[i])
        outs.append(ol.oracle_forward(prob, schema, n[i], net, X))
    return np.stack(outs)


def test_transform_order_matches_reference(fnb):
    prob = ol.Problem(16, 60, [0, 1, 2], [3])
    schema = ol.RICH
    nodes, conns = ol.random_genomes(71, schema, 300, 16, 60)
    eng = _engine(fnb, prob, schema)
    order, cnt = eng.transform(nodes, conns)
    for i in range(nodes.shape[0]):
        r = _ref_transform(prob, schema, nodes[i], conns[i])
        assert r["status"] == 0
        assert cnt[i] == r["order_count"]
        np.testing.assert_array_equal(order[i], r["order"])


@pytest.mark.parametrize("variant", ["wide_keys", "duplicate_rows"])
def test_transform_key_paths_match_reference(fnb, variant):
    """K1's rank keys are packed into 32 bits unless a key leaves [-2^23,
    2^23 - 1) (wide path), and its key -> row hash keeps the LOWEST row of a
    duplicated key (network.hpp:57-63): order and outputs against the reference."""
    prob = ol.Problem(16, 60, [0, 1, 2], [3])
    schema = ol.RICH
    nodes, conns = ol.random_genomes(2718, schema, 120, 16, 60)
    rng = np.random.default_rng(5)
    if variant == "wide_keys":
        for a in (nodes[..., 0], conns[..., 0], conns[..., 1]):
            a[a >= 4] += float(1 << 24)
    else:
        for i in range(nodes.shape[0]):
            live = np.where(~np.isnan(nodes[i, :, 0]))[0]
            empty = np.where(np.isnan(nodes[i, :, 0]))[0]
            if len(empty) and len(live) > 4:
                nodes[i, empty[rng.integers(len(empty))]] = nodes[i, live[4 + rng.integers(len(live) - 4)]]
    eng = _engine(fnb, prob, schema)
    order, cnt = eng.transform(nodes, conns)
    X = rng.uniform(-2, 2, size=(8, 3))
    want = _ref_forward(prob, schema, nodes, conns, X)
    got = eng.batch_forward(nodes, conns, X).values
    for i in range(nodes.shape[0]):
        r = _ref_transform(prob, schema, nodes[i], conns[i])
        assert r["status"] == 0
        assert cnt[i] == r["order_count"]
        np.testing.assert_array_equal(order[i], r["order"])
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("kind", ["cycle", "selfloop", "dangling", "bad_act", "bad_agg", "missing_output",
                                  "dup_pair"])
def test_transform_errors_match_reference(fnb, kind):
    from test_oracle_vs_ref import _corrupt
    prob = ol.Problem(16, 60, [0, 1, 2], [3])
    schema = ol.RICH
    nodes, conns = ol.random_genomes(5150, schema, 40, 16, 60)
    rng = np.random.default_rng(11)
    eng = _engine(fnb, prob, schema)
    for i in range(0, 40, 4):
        n, c = _corrupt(nodes[i], conns[i], rng, kind)
        r = _ref_transform(prob, schema, n, c)
        # the failing genome sits after a valid one: lowest-index error wins
        pn = np.stack([nodes[i + 1], n, nodes[i + 2]])
        pc = np.stack([conns[i + 1], c, conns[i + 2]])
        if r["status"] == 0:
            eng.transform(pn, pc)
            continue
        with pytest.raises(fnb.FlatneatError) as ei:
            eng.transform(pn, pc)
        assert ei.value.status == r["status"]
        assert ei.value.index == 1
        assert str(ei.value) == r["msg"], (kind, str(ei.value), r["msg"])


@pytest.mark.parametrize("seed,limits,schema_name", [
    (1312, (16, 60), "rich"), (90210, (50, 100), "rich"), (7, (20, 80), "tanh")])
def test_batch_forward_matches_reference(fnb, seed, limits, schema_name):
    schema = ol.RICH if schema_name == "rich" else ol.SchemaSpec()
    prob = ol.Problem(limits[0], limits[1], [0, 1, 2], [3])
    nodes, conns = ol.random_genomes(seed, schema, 200, *limits)
    rng = np.random.default_rng(seed)
    for B in (1, 4, 37, 300):
        X = rng.uniform(-2, 2, size=(B, 3))
        want = _ref_forward(prob, schema, nodes, conns, X)
        got = _engine(fnb, prob, schema).batch_forward(nodes, conns, X).values
        np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("act", ["tanh", "sigmoid", "identity", "relu"])
def test_single_activation_sum_kernels(fnb, act):
    """The {act},{sum} K2 instantiations (forward.cu) against the reference,
    and bit for bit against the generic kernel (a two-function schema whose
    first entries are the same functions, so the genomes mean the same).
    Bounded activations (tanh, sigmoid) leave pad-slot operand registers
    stale, unbounded ones zero them: with weights scaled by 1e20 the FP32
    identity / relu values overflow to +-inf (and inf - inf to NaN), where a
    stale inf under a pad slot's zero weight would turn an inf into NaN."""
    schema = ol.SchemaSpec([act], ["sum"])
    other = "identity" if act != "identity" else "tanh"
    generic = ol.SchemaSpec([act, other], ["sum", "product"])
    prob = ol.Problem(24, 96, [0, 1, 2], [3])
    nodes, conns = ol.random_genomes(515, schema, 160, 24, 96)
    rng = np.random.default_rng(515)
    X = rng.uniform(-2, 2, size=(300, 3))
    eng, eng_g = _engine(fnb, prob, schema), _engine(fnb, prob, generic)
    want = _ref_forward(prob, schema, nodes, conns, X)
    got = eng.batch_forward(nodes, conns, X).values
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)
    assert np.array_equal(got, eng_g.batch_forward(nodes, conns, X).values)
    big = conns.copy()
    big[:, :, 3] *= 1e20
    got = eng.batch_forward(nodes, big, X).values
    ref = eng_g.batch_forward(nodes, big, X).values
    if act in ("identity", "relu"):
        assert not np.isfinite(ref).all()  # the case is exercised
    assert np.array_equal(got, ref, equal_nan=True), act


def test_forward_c2_shape_and_fitness(fnb):
    """Config-2 shape (N_max=64, C_max=256, fill 0.75) on a 512-genome slice."""
    from paper_2504_08339_b200.synthetic import regression_dataset, synthetic_population
    nodes, conns = synthetic_population(512, 64, 256, fill=0.75, n_act=5, n_agg=4, seed=3)
    schema = ol.RICH
    prob = ol.Problem(64, 256, [0, 1, 2, 3], [4])
    X, Y = regression_dataset(1024, seed=1)
    eng = _engine(fnb, prob, schema)
    got = eng.batch_forward(nodes, conns, X).values
    want = _ref_forward(prob, schema, nodes, conns, X)
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)
    fit = eng.evaluate(nodes, conns, X, Y, fnb.FIT_NEG_MSE)
    want_fit = -np.mean((Y[None, :, :] - want) ** 2, axis=(1, 2))
    np.testing.assert_allclose(fit, want_fit, rtol=RTOL, atol=0)
    fit2 = eng.evaluate(nodes, conns, X, Y, fnb.FIT_OFFSET_SSE, 4.0)
    np.testing.assert_allclose(fit2, 4.0 - np.sum((Y[None] - want) ** 2, axis=(1, 2)), rtol=RTOL)


def test_padding_invariance_bit_exact(fnb):
    """test_network.cpp:192-206: (50,100) vs (200,400) give identical outputs."""
    schema = ol.RICH
    small = ol.random_genomes(90210, schema, 60, 50, 100)
    big_n = np.full((60, 200, 5), np.nan)
    big_c = np.full((60, 400, 4), np.nan)
    big_n[:, :50] = small[0]
    big_c[:, :100] = small[1]
    X = np.random.default_rng(0).uniform(-2, 2, size=(64, 3))
    a = _engine(fnb, ol.Problem(50, 100, [0, 1, 2], [3]), schema).batch_forward(*small, X).values
    b = _engine(fnb, ol.Problem(200, 400, [0, 1, 2], [3]), schema).batch_forward(big_n, big_c, X).values
    assert np.array_equal(a, b)


def test_batch_equals_single(fnb):
    """test_network.cpp:131-159: batch result == per-genome forward, bit for bit."""
    schema = ol.RICH
    prob = ol.Problem(16, 60, [0, 1, 2], [3])
    nodes, conns = ol.random_genomes(1312, schema, 64, 16, 60)
    X = np.random.default_rng(1).uniform(-2, 2, size=(16, 3))
    eng = _engine(fnb, prob, schema)
    allv = eng.batch_forward(nodes, conns, X).values
    for p in range(0, 64, 7):
        one = eng.batch_forward(nodes[p:p + 1], conns[p:p + 1], X).values[0]
        assert np.array_equal(one, allv[p])


def test_non_finite_input_rejected(fnb):
    schema = ol.RICH
    prob = ol.Problem(16, 60, [0, 1, 2], [3])
    nodes, conns = ol.random_genomes(3, schema, 4, 16, 60)
    X = np.zeros((2, 3))
    X[1, 2] = np.nan
    with pytest.raises(fnb.FlatneatError) as ei:
        _engine(fnb, prob, schema).batch_forward(nodes, conns, X)
    assert ei.value.code == "non_finite_input" and str(ei.value) == "non_finite_input: input not finite"


def test_known_answers(fnb):
    """test_network.cpp:74-106: identity network, tanh(0.6), two-input sum."""
    schema = ol.SchemaSpec(["tanh", "sigmoid", "identity", "relu", "sin"], ["sum", "product", "max", "mean"])
    prob = ol.Problem(6, 8, [0], [1])
    n = np.full((1, 6, 5), np.nan)
    n[0, 0] = [0, 0.0, 1.0, 0, 2]
    n[0, 1] = [1, 0.1, 1.0, 0, 0]
    n[0, 2] = [2, 0.0, 1.0, 0, 0]
    c = np.full((1, 8, 4), np.nan)
    c[0, 0] = [0, 1, 1, 0.5]
    out = _engine(fnb, prob, schema).batch_forward(n, c, np.array([[1.0]])).values
    assert abs(out[0, 0, 0] - 0.5370495669980353) < 1e-6


def test_pipelined_host_path_chunks(fnb):
    """fnb_evaluate streams the population up in chunks (capi.cu evaluate_impl):
    3000 C2 genomes = 32 MB -> 4 chunks.  Fitness must equal the one-shot
    device path bit for bit (partition-invariant units), and a transform error
    in a late chunk must still be reported for the lowest failing genome."""
    import torch
    from paper_2504_08339_b200.synthetic import regression_dataset, synthetic_population
    P = 3000
    nodes, conns = synthetic_population(P, 64, 256, fill=0.75, seed=21)
    X, Y = regression_dataset(256, seed=2)
    prob = ol.Problem(64, 256, [0, 1, 2, 3], [4])
    eng = _engine(fnb, prob, ol.SchemaSpec())
    fit = eng.evaluate(nodes, conns, X, Y, fnb.FIT_NEG_MSE)
    dev = torch.device("cuda", 0)
    dn, dc = torch.from_numpy(nodes).to(dev), torch.from_numpy(conns).to(dev)
    nets = eng.alloc_nets(P)
    st = torch.cuda.current_stream()
    eng.transform_d(dn, dc, nets, st)
    f_d = torch.empty(P, dtype=torch.float64, device=dev)
    eng.forward_d(nets, P, torch.from_numpy(X.astype(np.float32)).to(dev),
                  torch.from_numpy(Y.astype(np.float32)).to(dev), fnb.FIT_NEG_MSE, 0.0, fitness=f_d, stream=st)
    torch.cuda.synchronize()
    assert np.array_equal(fit, f_d.cpu().numpy())
    # a dangling endpoint in genome 2900 (last chunk) and 2950: 2900 is reported
    bad_c = conns.copy()
    for g in (2950, 2900):
        bad_c[g, 0, 1] = 9999.0
    with pytest.raises(fnb.FlatneatError) as ei:
        eng.evaluate(nodes, bad_c, X, Y, fnb.FIT_NEG_MSE)
    assert ei.value.index == 2900 and ei.value.code == "dangling_endpoint"
    # the context recovers: the next call is clean and identical
    assert np.array_equal(eng.evaluate(nodes, conns, X, Y, fnb.FIT_NEG_MSE), fit)


# ---- BASELINE config 5 shapes (N_max=128, C_max=1024): K1 runs k_transform<4>,
# K2 the N=128 tile geometry --------------------------------

@pytest.mark.parametrize("schema_name", ["tanh", "rich"])
def test_transform_and_forward_c5_shape(fnb, schema_name):
    """C5 shape (pop 100k config: N128/C1024, fill 0.75) on a 96-genome slice:
    K1 order (k_transform<4>) bit-exact, K2 outputs within 1e-5, fitness."""
    from paper_2504_08339_b200.synthetic import regression_dataset, synthetic_population
    rich = schema_name == "rich"
    # {sum, max, mean}: a product over ~8 FP64 terms of N(0,1) weights stays far from FP32 overflow,
    # but not over the C5 fan-ins, where FP32 and FP64 saturate differently
    schema = ol.SchemaSpec(["tanh", "sigmoid", "identity", "relu", "sin"], ["sum", "max", "mean"]) if rich \
        else ol.SchemaSpec()
    nodes, conns = synthetic_population(96, 128, 1024, fill=0.75, n_act=5 if rich else 1, n_agg=3 if rich else 1,
                                        seed=55 if rich else 56)
    prob = ol.Problem(128, 1024, [0, 1, 2, 3], [4])
    eng = _engine(fnb, prob, schema)
    order, cnt = eng.transform(nodes, conns)
    for i in range(nodes.shape[0]):
        r = _ref_transform(prob, schema, nodes[i], conns[i])
        assert r["status"] == 0
        assert cnt[i] == r["order_count"]
        np.testing.assert_array_equal(order[i], r["order"])
    X, Y = regression_dataset(96, seed=5)
    want = _ref_forward(prob, schema, nodes, conns, X)
    got = eng.batch_forward(nodes, conns, X).values
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)
    fit = eng.evaluate(nodes, conns, X, Y, fnb.FIT_NEG_MSE)
    np.testing.assert_allclose(fit, -np.mean((Y[None] - want) ** 2, axis=(1, 2)), rtol=RTOL)


@pytest.mark.parametrize("kind", ["cycle", "selfloop", "dangling", "bad_act", "dup_pair"])
def test_transform_errors_c5_shape(fnb, kind):
    """k_transform<4> error paths, messages (the cycle path string) and the
    lowest failing genome at N128/C1024."""
    from test_oracle_vs_ref import _corrupt
    from paper_2504_08339_b200.synthetic import synthetic_population
    schema = ol.RICH
    prob = ol.Problem(128, 1024, [0, 1, 2, 3], [4])
    nodes, conns = synthetic_population(12, 128, 1024, fill=0.75, n_act=5, n_agg=4, seed=9)
    rng = np.random.default_rng(13)
    eng = _engine(fnb, prob, schema)
    for i in range(0, 12, 3):
        n, c = _corrupt(nodes[i], conns[i], rng, kind)
        r = _ref_transform(prob, schema, n, c)
        pn = np.stack([nodes[i + 1], nodes[i + 2], n, nodes[i]])
        pc = np.stack([conns[i + 1], conns[i + 2], c, conns[i]])
        if r["status"] == 0:
            eng.transform(pn, pc)
            continue
        with pytest.raises(fnb.FlatneatError) as ei:
            eng.transform(pn, pc)
        assert ei.value.status == r["status"] and ei.value.index == 2
        assert str(ei.value) == r["msg"], (kind, str(ei.value), r["msg"])


def test_c3_cppn_fitness_full_grid(fnb):
    """BASELINE config 3 at its real batch: 32 C2 networks queried at the full
    256 x 256 grid (B = 65,536 samples each), outputs and image-MSE fitness
    against the reference's batch_forward."""
    from paper_2504_08339_b200.synthetic import cppn_dataset, synthetic_population
    if not ol.ref_available():
        pytest.skip("needs oracle/_ref")
    nodes, conns = synthetic_population(32, 64, 256, fill=0.75, seed=33)
    X, Y = cppn_dataset(256)
    assert X.shape[0] == 65536
    schema = ol.SchemaSpec()
    prob = ol.Problem(64, 256, [0, 1, 2, 3], [4])
    st, bad, msg, want = ol.ref_batch_forward(prob, schema, nodes, conns, X, nthreads=os.cpu_count() or 4)
    assert st == 0, msg
    eng = _engine(fnb, prob, schema)
    got = eng.batch_forward(nodes, conns, X).values
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)
    fit = eng.evaluate(nodes, conns, X, Y, fnb.FIT_NEG_MSE)
    np.testing.assert_allclose(fit, -np.mean((Y[None] - want) ** 2, axis=(1, 2)), rtol=RTOL)
