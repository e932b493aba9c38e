"""SPEC's worked examples for the SPEC-only evolution module, asserted on the
frozen CPU restatement (oracle/evolution.c) AND on the device generation
loop (fnb_evolver_*, with injected populations and fitness).

The reference ships no code for these stages ("parity
unpinned"); its only golden vectors are the examples in SPEC.md:
  initialize_population
  speciate
  update_stagnation
  compute_spawn_counts
  reproduce
(the evolve examples, are in tests/test_gpu_evolve.py and
tests/test_evolve_run.py).  On the device side every example also checks
the device state against the restatement bit for bit.
"""
import math

import numpy as np
import pytest

import oracle_lib as ol

ACTS, AGGS = ["tanh", "sigmoid", "identity"], ["sum", "product"]
LIMITS = (24, 80)
PROB = ol.Problem(LIMITS[0], LIMITS[1], [0, 1, 2], [3])
SCHEMA = ol.SchemaSpec(ACTS, AGGS)
ZERO_MUT = dict(node_add=0.0, conn_add=0.0, node_delete=0.0, conn_delete=0.0, bias=(0.0, 1.0, 0.5, 0.0, 0.0),
                response=(1.0, 0.0, 0.0, 0.0, 0.0), weight=(0.0, 1.0, 0.5, 0.0, 0.0), activation_replace_rate=0.0,
                aggregation_replace_rate=0.0)


class OracleSide:
    """oracle/evolution.c through tests/oracle_lib.py."""

    def __init__(self, P, mutation=None, seed=5, **kw):
        cfg = ol.neat_cfg(P, mutation=ol.mut_cfg(**(mutation or {})), **kw)
        self.o = ol.OracleEvolution(PROB, SCHEMA, cfg, seed=seed)

    def init_population(self):
        self.o.init_population()

    def set_population(self, n, c):
        self.o.set_population(n, c)

    def step(self, fit):
        self.o.step(np.asarray(fit, dtype=np.float64))

    def species(self):
        v = self.o.species_view()
        v["species_of"] = self.o.species_of.copy()
        return v

    def population(self):
        return self.o.nodes.copy(), self.o.conns.copy()


class DeviceSide:
    """The device loop (fnb_evolver_*), with the restatement run beside it and
    compared bit for bit after every step."""

    _KW = dict(threshold="compatibility_threshold", survival="survival_threshold",
               spawn_rate="spawn_number_change_rate")

    def __init__(self, P, mutation=None, seed=5, **kw):
        import paper_2504_08339_b200 as fnb
        from paper_2504_08339_b200.evolve import Evolver, NeatConfig
        m = fnb.MutationConfig()
        for k, v in (mutation or {}).items():
            setattr(m, k, fnb.AttrMutation(*v) if isinstance(v, tuple) else v)
        self.eng = fnb.Engine(fnb.GenomeLimits(*LIMITS), [0, 1, 2], [3], fnb.AttributeSchema(ACTS, AGGS))
        self.ev = Evolver(self.eng, NeatConfig(pop_size=P, mutation=m, **{self._KW.get(k, k): v for k, v in kw.items()}),
                          seed=seed)
        self.shadow = OracleSide(P, mutation, seed, **kw)

    def init_population(self):
        self.ev.init_population()
        self.shadow.init_population()
        self._same()

    def set_population(self, n, c):
        self.ev.set_population(n, c)
        self.shadow.set_population(n, c)

    def step(self, fit):
        self.ev.set_fitness(fit)
        self.ev.step()
        self.shadow.step(fit)
        self._same()

    def species(self):
        return self.ev.species()

    def population(self):
        return self.ev.population()

    def _same(self):
        gn, gc = self.ev.population()
        wn, wc = self.shadow.population()
        assert np.array_equal(gn.view(np.uint64), wn.view(np.uint64))
        assert np.array_equal(gc.view(np.uint64), wc.view(np.uint64))
        a, b = self.ev.species(), self.shadow.species()
        assert a["count"] == b["count"]
        for k in ("ids", "spawn", "best", "stagnation"):
            np.testing.assert_array_equal(a[k], b[k], err_msg=k)
        if self.ev.state()[0] > 0:
            np.testing.assert_array_equal(a["species_of"], b["species_of"])
        assert self.ev.state()[1] == self.shadow.o.innov.next_key


def _device_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


SIDES = [pytest.param(OracleSide, id="oracle"), pytest.param(DeviceSide, id="device", marks=pytest.mark.gpu)]


@pytest.fixture(params=SIDES)
def side(request):
    if request.param is DeviceSide and not _device_available():
        pytest.skip("no CUDA device")
    return request.param


def _genomes(seed, count):
    return ol.random_genomes(seed, SCHEMA, count, *LIMITS)


def _stack(parts):
    return np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts])


def _repeat(n, c, i, k):
    return np.repeat(n[i:i + 1], k, axis=0), np.repeat(c[i:i + 1], k, axis=0)


# ---- initialize_population ---------------------------------------

def test_init_minimal_genomes(side):
    """I=3, O=1 -> 5 nodes, 4 conns per genome (3*1 + 1*1); same seed twice -> bit-identical."""
    a, b = side(40, seed=3), side(40, seed=3)
    a.init_population()
    b.init_population()
    n, c = a.population()
    assert np.all(np.sum(~np.isnan(n[:, :, 0]), axis=1) == 5)
    assert np.all(np.sum(~np.isnan(c[:, :, 0]), axis=1) == 4)
    assert np.all(c[~np.isnan(c[:, :, 0])][:, 2] == 1.0)  # dense ENABLED conns
    n2, c2 = b.population()
    assert np.array_equal(n.view(np.uint64), n2.view(np.uint64)) and np.array_equal(c.view(np.uint64), c2.view(np.uint64))


@pytest.mark.gpu
def test_init_pop_size_one_rejected():
    """pop_size = 1 is rejected by the config invariant."""
    if not _device_available():
        pytest.skip("no CUDA device")
    import paper_2504_08339_b200 as fnb
    from paper_2504_08339_b200.evolve import Evolver, NeatConfig
    eng = fnb.Engine(fnb.GenomeLimits(*LIMITS), [0, 1, 2], [3], fnb.AttributeSchema(ACTS, AGGS))
    with pytest.raises(fnb.FlatneatError) as ei:
        Evolver(eng, NeatConfig(pop_size=1), seed=0)
    assert ei.value.code == "config_error"


# ---- speciate ----------------------------------------------------------

def test_speciate_infinite_threshold_one_species(side):
    """threshold = +inf -> exactly one species."""
    s = side(60, threshold=math.inf)
    s.set_population(*_genomes(7, 60))
    s.step(np.arange(60, dtype=np.float64))
    sp = s.species()
    assert sp["count"] == 1 and np.all(sp["species_of"] == 0)


def test_speciate_zero_threshold_max_species_and_nearest(side):
    """threshold = 0 with all-distinct genomes -> species count = max_species,
    overflow assigned to the nearest representative (brute force of the rule)."""
    P, S = 40, 5
    n, c = _genomes(8, P)
    s = side(P, threshold=0.0, max_species=S)
    s.set_population(n, c)
    s.step(np.linspace(0.0, 1.0, P))
    sp = s.species()
    assert sp["count"] == S
    want = list(range(S))  # founders: the lowest unassigned indices, in order
    for i in range(S, P):
        d = [ol.distance(PROB, n[i], c[i], n[j], c[j]) for j in range(S)]
        want.append(int(np.argmin(d)))  # argmin = lowest id on ties
    np.testing.assert_array_equal(sp["species_of"], want)


def test_speciate_two_identical_subpopulations(side):
    """two identical sub-populations, threshold between intra (0) and inter
    distance -> exactly 2 species."""
    n, c = _genomes(9, 2)
    d = ol.distance(PROB, n[0], c[0], n[1], c[1])
    assert d > 0
    pop = _stack([_repeat(n, c, 0, 25), _repeat(n, c, 1, 25)])
    perm = np.random.default_rng(1).permutation(50)  # interleaved
    s = side(50, threshold=d / 2)
    s.set_population(pop[0][perm], pop[1][perm])
    s.step(np.arange(50, dtype=np.float64))
    sp = s.species()
    assert sp["count"] == 2
    first = perm[0] < 25
    np.testing.assert_array_equal(sp["species_of"], np.where((perm < 25) == first, 0, 1))


# ---- update_stagnation ------------------------------------------------------

def test_stagnation_improving_species_resets(side):
    """improving species -> counter 0."""
    s = side(40, threshold=math.inf)
    s.set_population(*_genomes(10, 40))
    for g in range(5):
        s.step(np.full(40, float(g)) + np.linspace(0, 0.5, 40))
        assert s.species()["stagnation"].tolist() == [0]


def test_stagnation_protected_by_species_elitism(side):
    """1 species stagnant 16 generations, species_elitism = 2 -> retained."""
    s = side(30, threshold=math.inf, max_stagnation=15, species_elitism=2)
    s.set_population(*_genomes(11, 30))
    for _ in range(17):  # generation 0 sets best-ever; 16 stagnant ones follow
        s.step(np.zeros(30))
    sp = s.species()
    assert sp["count"] == 1 and sp["stagnation"].tolist() == [16]


def test_stagnation_worst_of_three_removed(side):
    """3 species stagnant, species_elitism = 2 -> the worst one is removed.
    No mutation, so every species stays a set of identical genomes; fitness
    is a function of the genome (A: 3, B: 2, C: 1)."""
    n, c = _genomes(12, 3)
    dmin = min(ol.distance(PROB, n[i], c[i], n[j], c[j]) for i in range(3) for j in range(3) if i != j)
    s = side(30, threshold=dmin / 2, max_stagnation=2, species_elitism=2, genome_elitism=1, mutation=ZERO_MUT)
    s.set_population(*_stack([_repeat(n, c, 0, 10), _repeat(n, c, 1, 10), _repeat(n, c, 2, 10)]))
    value = {0: 3.0, 1: 2.0, 2: 1.0}

    def fitness():
        pn, _ = s.population()
        out = []
        for g in pn:
            k = [i for i in range(3) if np.array_equal(g.view(np.uint64), n[i].view(np.uint64))]
            assert len(k) == 1
            out.append(value[k[0]])
        return np.array(out)

    counts = []
    for _ in range(4):
        s.step(fitness())
        counts.append(int(s.species()["count"]))
    # gen 0 sets best-ever (counter 0), gens 1-2 count to 2, gen 3 reaches 3 > 2
    assert counts == [3, 3, 3, 2]
    sp = s.species()
    assert sp["ids"].tolist() == [0, 1] and sp["best"].tolist() == [3.0, 2.0]
    pn, _ = s.population()
    assert not any(np.array_equal(g.view(np.uint64), n[2].view(np.uint64)) for g in pn)


# ---- compute_spawn_counts ------------------------------------------------------

def test_spawn_identical_distributions_equal_split(side):
    """two species, identical fitness distributions, equal old sizes -> equal split."""
    n, c = _genomes(13, 2)
    d = ol.distance(PROB, n[0], c[0], n[1], c[1])
    s = side(20, threshold=d / 2)
    s.set_population(*_stack([_repeat(n, c, 0, 10), _repeat(n, c, 1, 10)]))
    f = np.arange(10, dtype=np.float64)
    s.step(np.concatenate([f, f]))
    assert s.species()["spawn"].tolist() == [10, 10]


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_spawn_counts_sum_to_pop_size(side, seed):
    """counts always sum to pop_size (random instances)."""
    rng = np.random.default_rng(seed)
    P = int(rng.integers(30, 90))
    s = side(P, threshold=float(rng.uniform(0.3, 1.5)), max_species=int(rng.integers(2, 9)),
             spawn_rate=float(rng.uniform(0.1, 1.0)), genome_elitism=int(rng.integers(0, 3)))
    s.set_population(*_genomes(100 + seed, P))
    for _ in range(3):
        s.step(rng.normal(size=P))
        assert int(np.sum(s.species()["spawn"])) == P


def test_spawn_clamp_old_100_rate_half(side):
    """one species with old size 100, target below 50, rate 0.5 -> new size 50.
    (Two species of 100, A holding the 100 lowest ranks: target_A = 200 *
    49.5 / 199 = 49.75, clamped to 100 - round(0.5 * 100) = 50; B's 150.25 is
    clamped to 150, so the clamped sizes already sum to pop_size.)"""
    n, c = _genomes(14, 2)
    d = ol.distance(PROB, n[0], c[0], n[1], c[1])
    s = side(200, threshold=d / 2, spawn_rate=0.5)
    s.set_population(*_stack([_repeat(n, c, 0, 100), _repeat(n, c, 1, 100)]))
    s.step(np.arange(200, dtype=np.float64))
    assert s.species()["spawn"].tolist() == [50, 150]


# ---- reproduce ------------------------------------------------------------------------

def test_reproduce_singleton_species_spawn_three(side):
    """species of size 1, spawn 3, elitism 1 -> 1 elite copy + 2 mutated
    self-crossovers.  Population [A, B, B, B], fitness [10, 1, 2, 3]: A's
    mid-rank mean is 1, B's 1/3, so A's target is 3; rate 2 lets size 1 reach it."""
    n, c = _genomes(15, 2)
    d = ol.distance(PROB, n[0], c[0], n[1], c[1])
    s = side(4, threshold=d / 2, max_species=2, genome_elitism=1, spawn_rate=2.0, mutation=dict(ZERO_MUT, weight=(0.0, 1.0, 0.5, 1.0, 0.0)))
    pn, pc = _stack([_repeat(n, c, 0, 1), _repeat(n, c, 1, 3)])
    s.set_population(pn, pc)
    s.step(np.array([10.0, 1.0, 2.0, 3.0]))
    sp = s.species()
    assert sp["count"] == 2 and sp["spawn"].tolist() == [3, 1]
    qn, qc = s.population()
    assert np.array_equal(qn[0].view(np.uint64), n[0].view(np.uint64))  # the elite
    assert np.array_equal(qc[0].view(np.uint64), c[0].view(np.uint64))
    for k in (1, 2):  # self-crossover keeps A's structure; weight mutation rate 1 changes every weight
        np.testing.assert_array_equal(qn[k][:, 0], n[0][:, 0])
        np.testing.assert_array_equal(qc[k][:, :3], c[0][:, :3])
        live = ~np.isnan(c[0][:, 0])
        assert np.all(qc[k][live, 3] != c[0][live, 3])
    assert np.array_equal(qc[3].view(np.uint64), c[1].view(np.uint64))  # B's elite
    if side is OracleSide:
        pa, pb = s.o.last_parents
        assert pa[1] == pb[1] == 0 and pa[2] == pb[2] == 0


def test_reproduce_zero_mutation_full_elitism_identity(side):
    """all mutation probabilities 0, elitism = size -> next generation identical."""
    P = 30
    s = side(P, threshold=math.inf, max_species=1, genome_elitism=P, mutation=ZERO_MUT)
    n, c = _genomes(16, P)
    s.set_population(n, c)
    s.step(np.zeros(P))  # equal fitness: elites in index order
    qn, qc = s.population()
    assert np.array_equal(qn.view(np.uint64), n.view(np.uint64)) and np.array_equal(qc.view(np.uint64), c.view(np.uint64))


def test_reproduce_parent_pool_top_two(side):
    """survival_threshold 0.2, species size 10 -> parent pool = top 2: with no
    mutation and structurally identical genomes, every child's attributes
    come from the two fittest genomes."""
    P = 10
    base_n, base_c = _genomes(17, 1)
    n, c = _repeat(base_n, base_c, 0, P)
    n, c = n.copy(), c.copy()
    rng = np.random.default_rng(17)
    live_n, live_c = ~np.isnan(n[:, :, 0]), ~np.isnan(c[:, :, 0])
    n[:, :, 1] = np.where(live_n, rng.normal(size=live_n.shape), np.nan)
    c[:, :, 3] = np.where(live_c, rng.normal(size=live_c.shape), np.nan)
    fit = rng.permutation(P).astype(np.float64)
    top2 = np.argsort(-fit)[:2]
    s = side(P, threshold=math.inf, genome_elitism=0, survival=0.2, mutation=ZERO_MUT)
    s.set_population(n, c)
    s.step(fit)
    qn, qc = s.population()
    for k in range(P):
        for r in np.flatnonzero(live_n[0]):
            assert qn[k, r, 1] in (n[top2[0], r, 1], n[top2[1], r, 1])
        for r in np.flatnonzero(live_c[0]):
            assert qc[k, r, 3] in (c[top2[0], r, 3], c[top2[1], r, 3])
    if side is OracleSide:
        pa, pb = s.o.last_parents
        assert set(pa.tolist()) | set(pb.tolist()) <= set(top2.tolist())
