"""GPU parity for the device RNG (philox.cuh), K3 distance and K5 crossover.

All three are bit-exact against the reference (oracle/_ref when present,
else the pinned C restatement)."""
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


def _engine(fnb, prob, schema):
    return fnb.Engine(fnb.GenomeLimits(prob.max_nodes, prob.max_conns), prob.input_keys, prob.output_keys,
                      fnb.AttributeSchema(list(schema.activations), list(schema.aggregations)))


def test_host_key_tree_matches_reference(fnb):
    from paper_2504_08339_b200.api import key_seed, key_split
    for seed in (0, 1, 42, 2**40 + 3):
        k = key_seed(seed)
        assert np.array_equal(k, ol.key_words(ol.key_seed(seed)))
        for i in (0, 5, 2**33 + 1):
            assert np.array_equal(key_split(k, i), ol.key_words(ol.key_split(ol.key_seed(seed), i)))


def test_device_streams_match_reference(fnb):
    import torch
    prob = ol.Problem(8, 8, [0], [1])
    eng = _engine(fnb, prob, ol.SchemaSpec())
    root = ol.key_seed(7)
    keys = np.stack([ol.key_words(ol.key_split(root, i)) for i in range(64)])
    dk = torch.from_numpy(keys.view(np.int32)).cuda()
    # split_keys_d reproduces RngKey::split on the device
    sk = eng.split_keys_d(ol.key_words(root), 0, 64).cpu().numpy().view(np.uint32)
    assert np.array_equal(sk, keys)
    u = eng.stream_draws_d(dk, 33, kind=0).cpu().numpy().view(np.uint64)
    b = eng.stream_draws_d(dk, 33, kind=2, n=3 * 2**61).cpu().numpy().view(np.uint64)
    f = eng.stream_draws_d(dk, 33, kind=1).cpu().numpy().view(np.float64)
    for i in range(64):
        s = ol.stream(ol.key_from_words(keys[i]))
        assert [ol.oracle().fo_next_u64(ol.C.byref(s)) for _ in range(33)] == [int(x) for x in u[i]]
        s = ol.stream(ol.key_from_words(keys[i]))
        assert [ol.oracle().fo_below(ol.C.byref(s), 3 * 2**61) for _ in range(33)] == [int(x) for x in b[i]]
        s = ol.stream(ol.key_from_words(keys[i]))
        assert [ol.oracle().fo_uniform(ol.C.byref(s)) for _ in range(33)] == list(f[i])


def _ref_normals(keys, n_draws):
    """RngStream::normal(0, 1) (rng.hpp:111-116) of the REFERENCE with this
    host's glibc, n_draws per key, threaded over keys (ctypes drops the GIL)."""
    from concurrent.futures import ThreadPoolExecutor
    lib = ol.ref() if ol.ref_available() else None
    out = np.empty((keys.shape[0], n_draws))

    def one(i):
        k = np.ascontiguousarray(keys[i], dtype=np.uint32)
        row = out[i]
        if lib is not None:
            lib.fr_stream_draws(k.ctypes.data_as(ol.C.POINTER(ol.C.c_uint32)), 2, n_draws, ol.C.c_double(0.0),
                                ol.C.c_double(1.0), None, row.ctypes.data_as(ol.C.POINTER(ol.C.c_double)))
        else:
            s = ol.stream(ol.key_from_words(keys[i]))
            for d in range(n_draws):
                row[d] = ol.oracle().fo_normal(ol.C.byref(s), 0.0, 1.0)

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        list(ex.map(one, range(keys.shape[0])))
    return out


def test_device_normals_match_reference_1e8(fnb):
    """H1 on the device: 1.0e8 RngStream::normal draws (4 chunks of 1024 keys
    x 24,415 draws) are bit-identical to the reference's host normals, whose
    log / cos come from this box's glibc."""
    import torch
    if not ol.ref_available():
        pytest.skip("needs oracle/_ref (the reference's own RngStream::normal)")
    prob = ol.Problem(8, 8, [0], [1])
    eng = _engine(fnb, prob, ol.SchemaSpec())
    n_draws, total = 24415, 0
    for chunk in range(4):
        root = ol.key_split(ol.key_seed(2025), chunk)
        keys = np.stack([ol.key_words(ol.key_split(root, i)) for i in range(1024)])
        dk = torch.from_numpy(keys.view(np.int32)).cuda()
        got = eng.stream_draws_d(dk, n_draws, kind=3).cpu().numpy().view(np.float64)
        want = _ref_normals(keys, n_draws)
        bad = np.flatnonzero(got.view(np.uint64) != want.view(np.uint64))
        assert bad.size == 0, f"chunk {chunk}: {bad.size} mismatches, first at {bad[:4]}"
        total += got.size
    assert total >= 10**8


@pytest.mark.parametrize("seed,limits", [(31, (20, 80)), (2024, (64, 256))])
def test_distance_bit_exact(fnb, seed, limits):
    schema = ol.SchemaSpec(["tanh", "identity", "sigmoid"], ["sum", "product"])
    prob = ol.Problem(limits[0], limits[1], [0, 1, 2], [3])
    nodes, conns = ol.random_genomes(seed, schema, 120, *limits)
    # representatives: genomes from the same pool plus mutated relatives
    cfg = ol.mut_cfg(node_add=0.5, conn_add=0.5, node_delete=0.2, conn_delete=0.2)
    keys = np.stack([ol.key_words(ol.key_split(ol.key_seed(seed), i)) for i in range(120)])
    st, _, _, mn, mc = ol.mutate_population(prob, schema, nodes, conns, keys, cfg, 1000)
    assert st == 0
    reps_n = np.concatenate([nodes[:5], mn[5:10]])
    reps_c = np.concatenate([conns[:5], mc[5:10]])
    got = _engine(fnb, prob, schema).distance(mn, mc, reps_n, reps_c)
    use_ref = ol.ref_available()
    for p in range(mn.shape[0]):
        for s in range(reps_n.shape[0]):
            want = ol.distance(prob, mn[p], mc[p], reps_n[s], reps_c[s], use_ref=use_ref)
            assert got[p, s] == want, (p, s, got[p, s], want)


def test_distance_more_node_steps_than_conn_steps(fnb):
    """N_max = 100, C_max = 40: four 32-row node steps against two connection
    steps, node rows scattered so the last node step holds genes."""
    schema = ol.SchemaSpec(["tanh", "identity"], ["sum"])
    prob = ol.Problem(100, 40, [0, 1, 2], [3])
    nodes, conns = ol.random_genomes(404, schema, 60, 100, 40)
    rng = np.random.default_rng(404)
    for i in range(nodes.shape[0]):
        nodes[i] = nodes[i][rng.permutation(100)]
    reps_n, reps_c = nodes[:4].copy(), conns[:4].copy()
    got = _engine(fnb, prob, schema).distance(nodes, conns, reps_n, reps_c)
    use_ref = ol.ref_available()
    for p in range(nodes.shape[0]):
        for s in range(reps_n.shape[0]):
            want = ol.distance(prob, nodes[p], conns[p], reps_n[s], reps_c[s], use_ref=use_ref)
            assert got[p, s] == want, (p, s, got[p, s], want)


def test_distance_known_answer(fnb):
    """test_ops.cpp:244-255: identical genomes -> 0, one extra node -> 1/5."""
    schema = ol.SchemaSpec(["tanh", "identity"], ["sum"])
    prob = ol.Problem(8, 8, [0], [1])
    n = np.full((1, 8, 5), np.nan)
    for k in range(4):
        n[0, k] = [k, 0.0, 1.0, 0, 0]
    c = np.full((1, 8, 4), np.nan)
    n2 = n.copy()
    n2[0, 4] = [9, 0.0, 1.0, 0, 0]
    eng = _engine(fnb, prob, schema)
    assert eng.distance(n, c, n, c)[0, 0] == 0.0
    assert eng.distance(n, c, n2, c)[0, 0] == 1.0 / 5.0


@pytest.mark.parametrize("seed,limits", [(88, (20, 80)), (5, (64, 256))])
def test_crossover_bit_exact(fnb, seed, limits):
    schema = ol.SchemaSpec(["tanh", "identity"], ["sum"])
    prob = ol.Problem(limits[0], limits[1], [0, 1, 2], [3])
    nodes, conns = ol.random_genomes(seed, schema, 80, *limits)
    # related parents (shared markers) from a mutation step
    keys = np.stack([ol.key_words(ol.key_split(ol.key_seed(seed + 1), i)) for i in range(80)])
    st, _, _, mn, mc = ol.mutate_population(prob, schema, nodes, conns, keys, ol.mut_cfg(), 500)
    assert st == 0
    ck = np.stack([ol.key_words(ol.key_split(ol.key_seed(9), t)) for t in range(80)])
    cn, cc = _engine(fnb, prob, schema).crossover(nodes, conns, mn, mc, ck)
    use_ref = ol.ref_available()
    for t in range(80):
        wn, wc = ol.crossover(prob, nodes[t], conns[t], mn[t], mc[t], ol.key_from_words(ck[t]), use_ref=use_ref)
        np.testing.assert_array_equal(cn[t], wn)
        np.testing.assert_array_equal(cc[t], wc)


def test_crossover_identical_parents(fnb):
    """test_ops.cpp:198-204: identical parents give an identical child."""
    schema = ol.SchemaSpec(["tanh", "identity"], ["sum"])
    prob = ol.Problem(20, 80, [0, 1, 2], [3])
    nodes, conns = ol.random_genomes(3, schema, 16, 20, 80)
    ck = np.stack([ol.key_words(ol.key_split(ol.key_seed(1), t)) for t in range(16)])
    cn, cc = _engine(fnb, prob, schema).crossover(nodes, conns, nodes, conns, ck)
    np.testing.assert_array_equal(cn, nodes)
    np.testing.assert_array_equal(cc, conns)


def test_cpp_dropin_header(fnb):
    """include/flatneat/gpu.hpp used with the reference's own C++ types and
    functions (tests/cpp/test_gpu_hpp.cpp, built by __graft_entry__.build())."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(__file__), "cpp", "_bin", "test_gpu_hpp")
    if not os.path.exists(exe):
        pytest.skip("test_gpu_hpp not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "gpu.hpp parity ok" in r.stdout, r.stdout + r.stderr


def test_distance_union_tables_edge_cases(fnb):
    """K3's merged representative tables (distance.cu): 32 representatives
    (the ABI maximum), C5 row limits, and duplicated markers -- a repeated
    connection / node key in a representative resolves to its FIRST row, as
    the reference's linear find_conn / find_node do (genome.hpp:195-210)."""
    from paper_2504_08339_b200.synthetic import synthetic_population
    schema = ol.SchemaSpec()
    prob = ol.Problem(128, 1024, [0, 1, 2, 3], [4])
    nodes, conns = synthetic_population(72, 128, 1024, fill=0.75, seed=77)
    reps_n, reps_c = nodes[40:72].copy(), conns[40:72].copy()
    gn, gc = nodes[:40].copy(), conns[:40].copy()
    # share markers: genome i copies half of rep (i % 32)'s connections
    for i in range(40):
        gc[i, :384] = reps_c[i % 32, :384]
        gc[i, :384, 3] += 0.25 * i
    # duplicates: rep 3 repeats row 10 with another weight after its rows;
    # genome 5 repeats its own row 7; rep 6 repeats a node key
    reps_c[3, 900] = reps_c[3, 10]
    reps_c[3, 900, 3] = 123.0
    gc[5, 901] = gc[5, 7]
    reps_n[6, 120] = reps_n[6, 9]
    reps_n[6, 120, 1] = -7.0
    got = _engine(fnb, prob, schema).distance(gn, gc, reps_n, reps_c)
    use_ref = ol.ref_available()
    for p in range(gn.shape[0]):
        for s in range(32):
            want = ol.distance(prob, gn[p], gc[p], reps_n[s], reps_c[s], use_ref=use_ref)
            assert got[p, s] == want, (p, s, got[p, s], want)
    # one representative, and an empty population slice, go through the same path
    one = _engine(fnb, prob, schema).distance(gn[:3], gc[:3], reps_n[:1], reps_c[:1])
    for p in range(3):
        assert one[p, 0] == ol.distance(prob, gn[p], gc[p], reps_n[0], reps_c[0], use_ref=use_ref)


@pytest.mark.parametrize("variant", ["compact", "full_codes", "full_species"])
def test_distance_image_formats(fnb, variant):
    """K3's image formats (distance.cu): the compact one (S <= 16, small-integer
    agg / act codes) and the full one -- forced by a representative whose agg
    is not a small integer, or by more than 16 representatives -- give the
    reference's distances bit for bit, including genomes whose own agg / act
    are not small integers (code 0xFFFF)."""
    from paper_2504_08339_b200.synthetic import synthetic_population
    schema = ol.SchemaSpec(["tanh", "identity", "sigmoid"], ["sum", "product"])
    prob = ol.Problem(64, 256, [0, 1, 2, 3], [4])
    nodes, conns = synthetic_population(60, 64, 256, fill=0.75, n_act=3, n_agg=2, seed=404)
    S = 20 if variant == "full_species" else 10
    reps_n, reps_c = nodes[40:40 + S].copy(), conns[40:40 + S].copy()
    gn, gc = nodes[:40].copy(), conns[:40].copy()
    for i in range(40):  # shared markers with perturbed weights / attributes
        gc[i, :100] = reps_c[i % S, :100]
        gc[i, :100, 3] *= 1.0 + 0.01 * i
        gn[i, 5:20, 3] = (gn[i, 5:20, 3] + i) % 2
    gn[3, 7, 3] = 1.5        # a genome agg that is not a small integer
    gn[4, 8, 4] = 70000.0    # ... and a large act
    gn[5, 9, 3] = -0.0       # -0.0 == 0.0
    if variant == "full_codes":
        reps_n[2, 6, 3] = 2.5
    got = _engine(fnb, prob, schema).distance(gn, gc, reps_n, reps_c)
    use_ref = ol.ref_available()
    for p in range(gn.shape[0]):
        for s in range(S):
            want = ol.distance(prob, gn[p], gc[p], reps_n[s], reps_c[s], use_ref=use_ref)
            assert got[p, s] == want, (variant, p, s, got[p, s], want)


def test_crossover_c5_shape_bit_exact(fnb):
    """K5 at BASELINE config 5 shapes (N128/C1024, fill 0.75): 96 children of
    related parents (the reference's mutate of each parent) against the
    reference's crossover, bit for bit."""
    from paper_2504_08339_b200.synthetic import synthetic_population
    schema = ol.SchemaSpec()
    prob = ol.Problem(128, 1024, [0, 1, 2, 3], [4])
    nodes, conns = synthetic_population(96, 128, 1024, fill=0.75, seed=61)
    keys = np.stack([ol.key_words(ol.key_split(ol.key_seed(62), i)) for i in range(96)])
    use_ref = ol.ref_available()
    st, _, _, mn, mc = ol.mutate_population(prob, schema, nodes, conns, keys,
                                            ol.mut_cfg(node_add=0.5, conn_add=0.5, node_delete=0.1), 500,
                                            use_ref=use_ref)
    assert st == 0
    ck = np.stack([ol.key_words(ol.key_split(ol.key_seed(63), t)) for t in range(96)])
    # both argument orders: the child takes the FIT parent's structure
    for a_n, a_c, b_n, b_c in ((nodes, conns, mn, mc), (mn, mc, nodes, conns)):
        cn, cc = _engine(fnb, prob, schema).crossover(a_n, a_c, b_n, b_c, ck)
        for t in range(96):
            wn, wc = ol.crossover(prob, a_n[t], a_c[t], b_n[t], b_c[t], ol.key_from_words(ck[t]), use_ref=use_ref)
            np.testing.assert_array_equal(cn[t], wn)
            np.testing.assert_array_equal(cc[t], wc)
