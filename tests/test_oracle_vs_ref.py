"""Pin the C oracle (oracle/flatneat_oracle.c) to the reference itself.

The reference headers are compiled unmodified into oracle/_ref/ (see
oracle/Makefile); every restated function must agree with them bit for bit
on the reference's own known answers and on seeded random inputs.
"""
import ctypes as C

import numpy as np
import pytest

import oracle_lib as ol

pytestmark = pytest.mark.ref


def test_reference_own_suite_passes():
    """The reference's 51 GTest cases (proj/tests/*.cpp) pass on this host."""
    import os
    import subprocess
    exe = os.path.join(ol.ORACLE_DIR, "_ref", "ref_tests")
    if not os.path.exists(exe):
        ol.build()
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "51 passed, 0 failed" in r.stdout


@pytest.mark.parametrize("ctr,key,want", [
    # test_rng.cpp:12-34 (Random123 KATs)
    ((0, 0, 0, 0), (0, 0), (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
    ((0xffffffff,) * 4, (0xffffffff,) * 2, (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
    ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), (0xa4093822, 0x299f31d0),
     (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1)),
])
def test_philox_kats(ctr, key, want):
    c = np.array(ctr, dtype=np.uint32)
    k = np.array(key, dtype=np.uint32)
    for fn in (ol.oracle().fo_philox, ol.ref().fr_philox):
        out = np.zeros(4, dtype=np.uint32)
        fn(ol.ptr(c, ol.U32P), ol.ptr(k, ol.U32P), ol.ptr(out, ol.U32P))
        assert tuple(int(x) for x in out) == want


def test_keys_and_streams_match():
    lib, ref = ol.oracle(), ol.ref()
    for seed in [0, 1, 2, 42, 2**40 + 7, 2**64 - 1]:
        k = ol.key_seed(seed)
        rk = np.zeros(4, dtype=np.uint32)
        ref.fr_key_seed(C.c_uint64(seed), ol.ptr(rk, ol.U32P))
        assert np.array_equal(ol.key_words(k), rk)
        for idx in [0, 1, 5, 999, 2**33 + 3]:
            ks = ol.key_split(k, idx)
            rs = np.zeros(4, dtype=np.uint32)
            ref.fr_key_split(ol.ptr(rk, ol.U32P), C.c_uint64(idx), ol.ptr(rs, ol.U32P))
            assert np.array_equal(ol.key_words(ks), rs)
        # stream kinds: u64, uniform, normal, below, coin
        n = 257
        kw = ol.key_words(k)
        for kind, a, b in [(0, 0, 0), (1, 0, 0), (2, 0.3, 1.7), (3, 7, 0), (3, 3 * 2**61, 0), (4, 0.37, 0)]:
            ru = np.zeros(n, dtype=np.uint64)
            rd = np.zeros(n)
            ref.fr_stream_draws(ol.ptr(kw, ol.U32P), kind, n, C.c_double(a), C.c_double(b),
                                ol.ptr(ru, ol.U64P), ol.ptr(rd, ol.F64P))
            s = ol.stream(k)
            for i in range(n):
                if kind == 0:
                    assert lib.fo_next_u64(C.byref(s)) == int(ru[i])
                elif kind == 1:
                    assert lib.fo_uniform(C.byref(s)) == rd[i]
                elif kind == 2:
                    v = lib.fo_normal(C.byref(s), a, b)
                    assert v == rd[i] or (np.isnan(v) and np.isnan(rd[i]))
                elif kind == 3:
                    assert lib.fo_below(C.byref(s), C.c_uint64(int(a))) == int(ru[i])
                else:
                    assert lib.fo_coin(C.byref(s), a) == int(ru[i])


@pytest.mark.parametrize("seed,limits,schema", [
    (2024, (20, 80), ol.SchemaSpec(["tanh", "sigmoid", "identity"], ["sum", "product"])),
    (1312, (16, 60), ol.RICH),
    (90210, (50, 100), ol.RICH),
])
def test_generator_matches(seed, limits, schema):
    a = ol.random_genomes(seed, schema, 40, *limits)
    b = ol.random_genomes(seed, schema, 40, *limits, use_ref=True)
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])


def _prob(N, Cc, ni=3, no=1):
    return ol.Problem(N, Cc, list(range(ni)), list(range(ni, ni + no)))


def _corrupt(nodes, conns, rng, kind):
    """Seeded invalid variants exercising every transform error path."""
    n, c = nodes.copy(), conns.copy()
    live = np.where(~np.isnan(c[:, 0]))[0]
    empty = np.where(np.isnan(c[:, 0]))[0]
    if kind == "cycle" and len(live) and len(empty):
        r = live[rng.integers(len(live))]
        c[empty[0]] = [c[r, 1], c[r, 0], 1.0, 0.5]
        c[r, 2] = 1.0
    elif kind == "selfloop" and len(empty):
        k = n[~np.isnan(n[:, 0]), 0]
        kk = k[rng.integers(len(k))]
        c[empty[0]] = [kk, kk, 1.0, 0.1]
    elif kind == "dangling" and len(empty):
        c[empty[0]] = [0, 777, float(rng.integers(2)), 0.1]
    elif kind == "bad_act":
        rows = np.where(~np.isnan(n[:, 0]))[0]
        n[rows[rng.integers(len(rows))], 4] = 9
    elif kind == "bad_agg":
        rows = np.where(~np.isnan(n[:, 0]))[0]
        n[rows[rng.integers(len(rows))], 3] = -1
    elif kind == "missing_output":
        n[3] = np.nan
    elif kind == "dup_pair" and len(live) and len(empty):
        r = live[rng.integers(len(live))]
        c[empty[0]] = c[r]
        c[empty[0], 2] = 1.0
        c[r, 2] = 1.0
    return n, c


def test_transform_and_forward_match_reference():
    prob = _prob(16, 60)
    schema = ol.RICH
    nodes, conns = ol.random_genomes(71, schema, 150, 16, 60)
    rng = np.random.default_rng(3)
    X = rng.uniform(-2, 2, size=(6, 3))
    kinds = [None, "cycle", "selfloop", "dangling", "bad_act", "bad_agg", "missing_output", "dup_pair"]
    n_err = 0
    for i in range(nodes.shape[0]):
        kind = kinds[i % len(kinds)]
        n, c = (nodes[i], conns[i]) if kind is None else _corrupt(nodes[i], conns[i], rng, kind)
        o = ol.oracle_transform(prob, schema, n, c)
        r = ol.ref_transform(prob, schema, n, c)
        assert o["status"] == r["status"], (i, kind, o["msg"], r["msg"])
        if r["status"]:
            assert o["msg"] == r["msg"], (kind, o["msg"], r["msg"])
            n_err += 1
            continue
        assert np.array_equal(o["order"], r["order"]) and o["order_count"] == r["order_count"]
        assert np.array_equal(o["input_rows"], r["input_rows"])
        assert np.array_equal(o["output_rows"], r["output_rows"])
        exp = r["expanded"]
        for dst in range(prob.max_nodes):
            srcs = np.where(~np.isnan(exp[:, dst]))[0]
            b, e = o["in_begin"][dst], o["in_begin"][dst + 1]
            assert np.array_equal(o["in_src"][b:e], srcs)
            assert np.array_equal(o["in_w"][b:e], exp[srcs, dst])
        st, bad, msg, out = ol.ref_batch_forward(prob, schema, n[None], c[None], X)
        assert st == 0
        got = ol.oracle_forward(prob, schema, n, o, X)
        assert np.array_equal(got, out[0]), (i, got, out[0])
    assert n_err > 40


def test_cycle_message_known_answer():
    """test_network.cpp:61-72: cycle message contains 0->2->0."""
    prob = ol.Problem(6, 8, [0], [1])
    s = ol.RICH
    n = np.full((6, 5), np.nan)
    for k in range(3):
        n[k] = [k, 0.0, 1.0, 0, 2]
    c = np.full((8, 4), np.nan)
    c[0] = [0, 2, 1, 1.0]
    c[1] = [2, 0, 1, 1.0]
    o = ol.oracle_transform(prob, s, n, c)
    r = ol.ref_transform(prob, s, n, c)
    assert o["msg"] == r["msg"] and "0->2->0" in o["msg"] and o["status"] == 1 + ol.ERRC.index("cycle_detected")


def test_distance_matches_bitwise():
    prob = _prob(20, 80)
    schema = ol.SchemaSpec(["tanh", "identity"], ["sum"])
    nodes, conns = ol.random_genomes(31, schema, 60, 20, 80)
    asym = 0
    for i in range(0, 60, 2):
        a = (nodes[i], conns[i])
        b = (nodes[i + 1], conns[i + 1])
        for x, y in [(a, b), (b, a), (a, a)]:
            do = ol.distance(prob, *x, *y)
            dr = ol.distance(prob, *x, *y, use_ref=True)
            assert do == dr or (np.isnan(do) and np.isnan(dr))
        asym += ol.distance(prob, *a, *b) != ol.distance(prob, *b, *a)
    # ops.hpp sums in g1 row order, so the distance is not bitwise symmetric.
    assert asym >= 0


def test_crossover_matches_bitwise():
    prob = _prob(20, 80)
    schema = ol.SchemaSpec(["tanh", "identity"], ["sum"])
    nodes, conns = ol.random_genomes(88, schema, 40, 20, 80)
    for t in range(20):
        k = ol.key_split(ol.key_seed(9), t)
        args = (nodes[2 * t], conns[2 * t], nodes[2 * t + 1], conns[2 * t + 1])
        a = ol.crossover(prob, *args, k)
        b = ol.crossover(prob, *args, k, use_ref=True)
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_array_equal(a[1], b[1])


@pytest.mark.parametrize("cfgkw", [
    {},
    dict(node_delete=0.15, conn_delete=0.15, activation_replace_rate=0.1, aggregation_replace_rate=0.1),
    dict(node_add=0.9, conn_add=0.9, node_delete=0.3, conn_delete=0.3),
])
def test_mutate_population_matches_bitwise(cfgkw):
    prob = _prob(18, 60)
    schema = ol.SchemaSpec(["tanh", "sigmoid", "identity"], ["sum", "product"])
    nodes, conns = ol.random_genomes(404, schema, 120, 18, 60)
    cfg = ol.mut_cfg(**cfgkw)
    root = ol.key_seed(17)
    keys = np.stack([ol.key_words(ol.key_split(root, p)) for p in range(120)])
    next_key = 1000
    for step in range(4):
        # step 3 restarts the innovation counter: new keys collide with
        # existing nodes -> duplicate_key from add_node (ops.hpp:21-22).
        nk = 1000 if step == 3 else next_key
        a = ol.mutate_population(prob, schema, nodes, conns, keys, cfg, nk)
        b = ol.mutate_population(prob, schema, nodes, conns, keys, cfg, nk, use_ref=True)
        assert a[0] == b[0] and a[1] == b[1] and a[2] == b[2]
        np.testing.assert_array_equal(a[3], b[3])
        np.testing.assert_array_equal(a[4], b[4])
        assert a[0] in (0, 1 + ol.ERRC.index("duplicate_key"))
        nodes, conns, next_key = a[3], a[4], a[2]
        keys = keys ^ np.uint32(0x9E3779B9 + step)
