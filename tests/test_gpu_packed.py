"""The packed host transfer of fnb_evaluate / fnb_batch_forward (capi.cu
evaluate_impl, ctx_internal.cuh pack_genomes, K1's kPk instantiation): the
host converts each chunk's FP64 rows into K1's transfer rows and only those
cross PCIe.  Every result -- fitness bits, outputs, error status, index and
message -- must equal the FP64-row path (fnb_set_host_transfer_packed(0)),
which tests/test_gpu_forward.py pins to the reference.
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
    yield m
    m._native.lib().fnb_set_host_transfer_packed(1)


def _engine(fnb, prob, schema):
    return fnb.Engine(fnb.GenomeLimits(prob.max_nodes, prob.max_conns), prob.input_keys, prob.output_keys,
                      fnb.AttributeSchema(list(schema.activations), list(schema.aggregations)))


def _both(fnb, f):
    """f() with packed transfer rows, then with the FP64 rows: (result or error) each."""
    out = []
    for packed in (1, 0):
        fnb._native.lib().fnb_set_host_transfer_packed(packed)
        try:
            out.append(("ok", f()))
        except fnb.FlatneatError as e:
            out.append(("err", (e.status, e.index, str(e))))
    fnb._native.lib().fnb_set_host_transfer_packed(1)
    return out


def _same(a, b):
    assert a[0] == b[0], (a, b)
    if a[0] == "err":
        assert a[1] == b[1]
    elif isinstance(a[1], np.ndarray):
        assert np.array_equal(a[1], b[1], equal_nan=True)
    else:
        assert np.array_equal(a[1].values, b[1].values, equal_nan=True)


@pytest.mark.parametrize("shape,P,schema_name", [((64, 256), 3000, "tanh"), ((16, 60), 200, "rich"),
                                                  ((128, 1024), 64, "tanh"), ((17, 61), 77, "rich")])
def test_packed_equals_fp64_rows(fnb, shape, P, schema_name):
    """Fitness and outputs bit-identical; 3000 C2 genomes span several chunks; odd
    N / C exercise the packed layout's alignment."""
    from paper_2504_08339_b200.synthetic import regression_dataset, synthetic_population
    schema = ol.RICH if schema_name == "rich" else ol.SchemaSpec()
    N, C = shape
    if schema_name == "rich":
        nodes, conns = ol.random_genomes(4242 + N, schema, P, N, C)
        ni = 3
    else:
        nodes, conns = synthetic_population(P, N, C, fill=0.75, seed=31)
        ni = 4
    prob = ol.Problem(N, C, list(range(ni)), [ni])
    eng = _engine(fnb, prob, schema)
    X, Y = regression_dataset(100, ni, 1, seed=3)
    r = _both(fnb, lambda: eng.evaluate(nodes, conns, X, Y, fnb.FIT_NEG_MSE))
    assert r[0][0] == "ok"
    _same(*r)
    _same(*_both(fnb, lambda: eng.batch_forward(nodes, conns, X)))


@pytest.mark.parametrize("kind", ["cycle", "selfloop", "dangling", "bad_act", "bad_agg", "missing_output",
                                  "dup_pair", "act_300", "agg_nan", "key_nan_conn_out", "wide_keys",
                                  "fractional_keys", "nan_weight", "neg_enabled"])
def test_packed_errors_and_edge_rows(fnb, kind):
    """Invalid and unusual rows: the same error (status, lowest index, message)
    or the same fitness through both transfer formats, and the reference's
    status and message for the errors it defines."""
    from test_oracle_vs_ref import _corrupt
    prob = ol.Problem(16, 60, [0, 1, 2], [3])
    schema = ol.RICH
    nodes, conns = ol.random_genomes(808, schema, 30, 16, 60)
    rng = np.random.default_rng(17)
    eng = _engine(fnb, prob, schema)
    X = np.random.default_rng(5).uniform(-1, 1, size=(40, 3))
    Y = np.random.default_rng(6).uniform(-1, 1, size=(40, 1))
    for i in range(0, 24, 6):
        n, c = nodes.copy(), conns.copy()
        g = i + 1
        live_n = np.where(~np.isnan(n[g, :, 0]))[0]
        live_c = np.where(~np.isnan(c[g, :, 0]))[0]
        if kind in ("cycle", "selfloop", "dangling", "bad_act", "bad_agg", "missing_output", "dup_pair"):
            n[g], c[g] = _corrupt(n[g], c[g], rng, kind)
        elif kind == "act_300":  # beyond the packed byte: the whole call falls back to the FP64 rows
            n[g, live_n[-1], 4] = 300.0
        elif kind == "agg_nan":
            n[g, live_n[-1], 3] = np.nan
        elif kind == "key_nan_conn_out":
            c[g, live_c[0], 1] = np.nan
        elif kind == "wide_keys":  # keys beyond 2^23: K1's 64-bit rank path
            hid = live_n[live_n >= 4]
            for r in hid:
                old = n[g, r, 0]
                new = old + 2.0 ** 30
                n[g, r, 0] = new
                c[g, c[g, :, 0] == old, 0] = new
                c[g, c[g, :, 1] == old, 1] = new
        elif kind == "fractional_keys":
            c[g, live_c[:3], 0] += 0.25
        elif kind == "nan_weight":
            c[g, live_c[:2], 3] = np.nan
            c[g, live_c[:2], 2] = 1.0
        elif kind == "neg_enabled":
            c[g, live_c[:4], 2] = -1.0
        r = _both(fnb, lambda: eng.evaluate(n, c, X, Y, fnb.FIT_NEG_MSE))
        _same(*r)
        rb = _both(fnb, lambda: eng.batch_forward(n, c, X))
        _same(*rb)
        ref = ol.ref_transform(prob, schema, n[g], c[g]) if ol.ref_available() else \
            ol.oracle_transform(prob, schema, n[g], c[g])
        if r[0][0] == "err" and r[0][1][1] == g and ref["status"] != 0 and kind not in ("agg_nan",):
            assert r[0][1][0] == ref["status"] and r[0][1][2] == ref["msg"], (kind, r[0][1], ref["msg"])


def test_packed_pinned_and_pageable(fnb):
    """Pinned and pageable host arrays give the same bits through the packer."""
    import torch
    from paper_2504_08339_b200.synthetic import regression_dataset, synthetic_population
    nodes, conns = synthetic_population(1500, 64, 256, fill=0.75, seed=8)
    X, Y = regression_dataset(64, seed=1)
    eng = _engine(fnb, ol.Problem(64, 256, [0, 1, 2, 3], [4]), ol.SchemaSpec())
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    a = eng.evaluate(nodes, conns, X, Y, fnb.FIT_NEG_MSE)
    b = eng.evaluate(pin(nodes), pin(conns), pin(X), pin(Y), fnb.FIT_NEG_MSE)
    fnb._native.lib().fnb_set_host_transfer_packed(0)
    c = eng.evaluate(nodes, conns, X, Y, fnb.FIT_NEG_MSE)
    fnb._native.lib().fnb_set_host_transfer_packed(1)
    assert np.array_equal(a, b) and np.array_equal(a, c)
