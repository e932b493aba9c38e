"""ctypes bindings to the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Two checkers live under oracle/ (see oracle/flatneat_oracle.h):
  * liboracle.so            -- the plain-C restatement of the reference path
                               plus the frozen SPEC evolution restatement;
  * _ref/libflatneat_ref.so -- the unmodified reference headers behind an
                               extern "C" shim (built in this container from
                               /root/reference; the .so travels to the GPU box).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import
this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")

ACT = {"identity": 0, "tanh": 1, "sigmoid": 2, "relu": 3, "sin": 4}
AGG = {"sum": 0, "product": 1, "max": 2, "mean": 3}
ERRC = ["unknown_function", "genome_full", "duplicate_key", "duplicate_conn",
        "dangling_endpoint", "key_not_found", "protected_node", "attr_out_of_range",
        "shape_mismatch", "corrupt_row", "cycle_detected", "non_finite_input",
        "non_finite_state", "empty_aggregation", "empty_dataset", "parse_error",
        "version_unsupported", "limits_too_small", "config_error", "eval_error"]

I32P = C.POINTER(C.c_int32)
U32P = C.POINTER(C.c_uint32)
U64P = C.POINTER(C.c_uint64)
F64P = C.POINTER(C.c_double)


class Shape(C.Structure):
    _fields_ = [("max_nodes", C.c_int), ("max_conns", C.c_int), ("num_inputs", C.c_int),
                ("num_outputs", C.c_int), ("input_keys", I32P), ("output_keys", I32P)]


class Schema(C.Structure):
    _fields_ = [("n_act", C.c_int), ("act", C.c_int * 8), ("n_agg", C.c_int), ("agg", C.c_int * 8),
                ("default_act", C.c_int), ("default_agg", C.c_int)]


class AttrMut(C.Structure):
    _fields_ = [("init_mean", C.c_double), ("init_std", C.c_double), ("mutate_power", C.c_double),
                ("mutate_rate", C.c_double), ("replace_rate", C.c_double)]


class MutCfg(C.Structure):
    _fields_ = [("node_add", C.c_double), ("node_delete", C.c_double), ("conn_add", C.c_double),
                ("conn_delete", C.c_double), ("bias", AttrMut), ("response", AttrMut),
                ("weight", AttrMut), ("activation_replace_rate", C.c_double),
                ("aggregation_replace_rate", C.c_double)]


class DistCfg(C.Structure):
    _fields_ = [("compatibility_disjoint", C.c_double), ("compatibility_homologous", C.c_double)]


class GenSpec(C.Structure):
    _fields_ = [("num_inputs", C.c_int), ("num_outputs", C.c_int), ("max_hidden", C.c_int),
                ("conn_prob", C.c_double), ("disabled_prob", C.c_double)]


class Key(C.Structure):
    _fields_ = [("w", C.c_uint32 * 4)]


class Stream(C.Structure):
    _fields_ = [("key", Key), ("block", C.c_uint64), ("buf", C.c_uint32 * 4), ("avail", C.c_int)]


class Net(C.Structure):
    _fields_ = [("order", I32P), ("order_count", C.c_int), ("in_begin", I32P), ("in_src", I32P),
                ("in_w", F64P), ("input_rows", I32P), ("output_rows", I32P), ("msg", C.c_char * 512)]


class NeatCfg(C.Structure):
    _fields_ = [("pop_size", C.c_int), ("max_species", C.c_int),
                ("compatibility_threshold", C.c_double), ("species_elitism", C.c_int),
                ("max_stagnation", C.c_int), ("genome_elitism", C.c_int),
                ("survival_threshold", C.c_double), ("spawn_number_change_rate", C.c_double),
                ("output_activation", C.c_int), ("mutation", MutCfg), ("distance", DistCfg)]


class Species(C.Structure):
    _fields_ = [("count", C.c_int), ("next_id", C.c_int), ("cap", C.c_int), ("nsz", C.c_size_t),
                ("csz", C.c_size_t), ("id", I32P), ("rep_nodes", F64P), ("rep_conns", F64P),
                ("best_fitness", F64P), ("stagnation", I32P), ("size", I32P), ("spawn", I32P)]


class InnovTable(C.Structure):
    _fields_ = [("next_key", C.c_int), ("count", C.c_int), ("cap", C.c_int), ("pairs", I32P)]


def ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def build() -> None:
    """Build liboracle.so (and _ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)


def _load(path: str) -> C.CDLL:
    if not os.path.exists(path):
        build()
    return C.CDLL(path)


_oracle = None
_ref = None


def oracle() -> C.CDLL:
    global _oracle
    if _oracle is None:
        lib = _load(os.path.join(ORACLE_DIR, "liboracle.so"))
        lib.fo_key_seed.restype = Key
        lib.fo_key_seed.argtypes = [C.c_uint64]
        lib.fo_key_split.restype = Key
        lib.fo_key_split.argtypes = [Key, C.c_uint64]
        lib.fo_next_u64.restype = C.c_uint64
        lib.fo_uniform.restype = C.c_double
        lib.fo_normal.restype = C.c_double
        lib.fo_normal.argtypes = [C.POINTER(Stream), C.c_double, C.c_double]
        lib.fo_below.restype = C.c_uint64
        lib.fo_below.argtypes = [C.POINTER(Stream), C.c_uint64]
        lib.fo_coin.argtypes = [C.POINTER(Stream), C.c_double]
        lib.fo_distance.restype = C.c_double
        lib.fo_crossover.argtypes = [C.POINTER(Shape), F64P, F64P, F64P, F64P, Key, F64P, F64P]
        lib.fo_mutate.argtypes = [C.POINTER(Shape), C.POINTER(Schema), F64P, F64P, Key,
                                  C.POINTER(MutCfg), C.POINTER(InnovTable)]
        lib.fo_plan_node_split.restype = C.c_int * 3
        lib.fo_initialize_population.argtypes = [C.POINTER(Shape), C.POINTER(Schema),
                                                 C.POINTER(NeatCfg), C.c_uint64, F64P, F64P]
        lib.fo_reproduce.argtypes = [C.POINTER(Shape), C.POINTER(Schema), C.POINTER(NeatCfg),
                                     F64P, F64P, F64P, I32P, C.POINTER(Species), C.c_uint64, C.c_int,
                                     C.POINTER(InnovTable), F64P, F64P, I32P, I32P]
        _oracle = lib
    return _oracle


def ref_available() -> bool:
    return os.path.exists(os.path.join(ORACLE_DIR, "_ref", "libflatneat_ref.so")) or \
        os.path.exists("/root/reference/proj/include/flatneat/network.hpp")


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        lib = _load(os.path.join(ORACLE_DIR, "_ref", "libflatneat_ref.so"))
        lib.fr_distance.restype = C.c_double
        _ref = lib
    return _ref


# ---------------------------------------------------------------------------
# Plain-Python configuration mirrors
# ---------------------------------------------------------------------------

@dataclass
class Problem:
    """Genome shape: limits plus input/output keys (genome.hpp:87-92, 151-152)."""
    max_nodes: int
    max_conns: int
    input_keys: list
    output_keys: list

    @property
    def num_inputs(self):
        return len(self.input_keys)

    @property
    def num_outputs(self):
        return len(self.output_keys)

    def c(self) -> Shape:
        ik = np.asarray(self.input_keys, dtype=np.int32)
        ok = np.asarray(self.output_keys, dtype=np.int32)
        s = Shape(self.max_nodes, self.max_conns, len(self.input_keys), len(self.output_keys),
                  ptr(ik, I32P), ptr(ok, I32P))
        s._keep = (ik, ok)  # the key arrays live as long as the struct
        return s

    def empty_pop(self, P: int):
        return (np.full((P, self.max_nodes, 5), np.nan), np.full((P, self.max_conns, 4), np.nan))


@dataclass
class SchemaSpec:
    activations: list = field(default_factory=lambda: ["tanh"])
    aggregations: list = field(default_factory=lambda: ["sum"])
    default_activation: int = 0
    default_aggregation: int = 0

    def c(self) -> Schema:
        s = Schema()
        s.n_act = len(self.activations)
        for i, a in enumerate(self.activations):
            s.act[i] = ACT[a]
        s.n_agg = len(self.aggregations)
        for i, a in enumerate(self.aggregations):
            s.agg[i] = AGG[a]
        s.default_act = self.default_activation
        s.default_agg = self.default_aggregation
        return s


RICH = SchemaSpec(["tanh", "sigmoid", "identity", "relu", "sin"], ["sum", "product", "max", "mean"])


def attr(init_mean, init_std, power, rate, replace):
    return AttrMut(init_mean, init_std, power, rate, replace)


def mut_cfg(**kw) -> MutCfg:
    """MutationConfig defaults (ops.hpp:125-135)."""
    m = MutCfg(0.2, 0.0, 0.4, 0.0, attr(0.0, 1.0, 0.5, 0.7, 0.1), attr(1.0, 0.0, 0.0, 0.0, 0.0),
               attr(0.0, 1.0, 0.5, 0.8, 0.1), 0.0, 0.0)
    for k, v in kw.items():
        if isinstance(v, tuple):
            v = attr(*v)
        setattr(m, k, v)
    return m


# ---------------------------------------------------------------------------
# Convenience wrappers
# ---------------------------------------------------------------------------

def key_seed(seed: int) -> Key:
    return oracle().fo_key_seed(seed)


def key_split(k: Key, i: int) -> Key:
    return oracle().fo_key_split(k, i)


def key_words(k: Key) -> np.ndarray:
    return np.array(list(k.w), dtype=np.uint32)


def key_from_words(w) -> Key:
    k = Key()
    for i in range(4):
        k.w[i] = int(w[i])
    return k


def stream(k: Key) -> Stream:
    s = Stream()
    oracle().fo_stream_init(C.byref(s), k)
    return s


def random_genomes(seed: int, schema: SchemaSpec, count: int, max_nodes: int, max_conns: int,
                   spec=(3, 1, 8, 0.5, 0.15), use_ref=False):
    """testgen::random_acyclic_genome x count from RngStream(RngKey(seed))."""
    nodes = np.full((count, max_nodes, 5), np.nan)
    conns = np.full((count, max_conns, 4), np.nan)
    sc = schema.c()
    gs = GenSpec(*spec)
    if use_ref:
        st = ref().fr_random_genomes(C.c_uint64(seed), C.byref(sc), C.byref(gs), count, max_nodes,
                                     max_conns, ptr(nodes, F64P), ptr(conns, F64P))
        assert st == 0, st
        return nodes, conns
    s = stream(key_seed(seed))
    for i in range(count):
        st = oracle().fo_random_acyclic_genome(C.byref(s), C.byref(sc), C.byref(gs), max_nodes,
                                                max_conns, ptr(nodes[i], F64P), ptr(conns[i], F64P))
        assert st == 0, st
    return nodes, conns


def oracle_transform(prob: Problem, schema: SchemaSpec, nodes: np.ndarray, conns: np.ndarray):
    N, Cc = prob.max_nodes, prob.max_conns
    order = np.full(N, -1, dtype=np.int32)
    in_begin = np.zeros(N + 1, dtype=np.int32)
    in_src = np.zeros(max(Cc, 1), dtype=np.int32)
    in_w = np.zeros(max(Cc, 1))
    irows = np.zeros(max(prob.num_inputs, 1), dtype=np.int32)
    orows = np.zeros(max(prob.num_outputs, 1), dtype=np.int32)
    net = Net(ptr(order, I32P), 0, ptr(in_begin, I32P), ptr(in_src, I32P), ptr(in_w, F64P),
              ptr(irows, I32P), ptr(orows, I32P))
    sh, sc = prob.c(), schema.c()
    nodes = np.ascontiguousarray(nodes, dtype=np.float64)
    conns = np.ascontiguousarray(conns, dtype=np.float64)
    st = oracle().fo_transform(C.byref(sh), C.byref(sc), ptr(nodes, F64P), ptr(conns, F64P), C.byref(net))
    return dict(status=st, msg=net.msg.decode(), order=order, order_count=net.order_count,
                in_begin=in_begin, in_src=in_src[:in_begin[N]], in_w=in_w[:in_begin[N]],
                input_rows=irows[:prob.num_inputs], output_rows=orows[:prob.num_outputs], _net=net,
                _keep=(order, in_begin, in_src, in_w, irows, orows))


def oracle_forward(prob: Problem, schema: SchemaSpec, nodes, net, X: np.ndarray) -> np.ndarray:
    """forward() of one transformed genome over B samples -> [B, O]."""
    sh, sc = prob.c(), schema.c()
    nodes = np.ascontiguousarray(nodes, dtype=np.float64)
    B = X.shape[0]
    out = np.zeros((B, prob.num_outputs))
    v = np.zeros(prob.max_nodes)
    X = np.ascontiguousarray(X, dtype=np.float64)
    for b in range(B):
        st = oracle().fo_forward(C.byref(sh), C.byref(sc), ptr(nodes, F64P), C.byref(net["_net"]),
                                 ptr(X[b], F64P), ptr(out[b], F64P), ptr(v, F64P))
        if st:
            raise RuntimeError(ERRC[st - 1])
    return out


def ref_transform(prob: Problem, schema: SchemaSpec, nodes, conns):
    N = prob.max_nodes
    order = np.full(N, -1, dtype=np.int32)
    cnt = C.c_int(0)
    expanded = np.zeros(N * N)
    irows = np.zeros(max(prob.num_inputs, 1), dtype=np.int32)
    orows = np.zeros(max(prob.num_outputs, 1), dtype=np.int32)
    msg = C.create_string_buffer(512)
    sh, sc = prob.c(), schema.c()
    nodes = np.ascontiguousarray(nodes, dtype=np.float64)
    conns = np.ascontiguousarray(conns, dtype=np.float64)
    st = ref().fr_transform(C.byref(sh), C.byref(sc), ptr(nodes, F64P), ptr(conns, F64P),
                            ptr(order, I32P), C.byref(cnt), ptr(expanded, F64P), ptr(irows, I32P),
                            ptr(orows, I32P), msg, C.c_size_t(512))
    return dict(status=st, msg=msg.value.decode(), order=order, order_count=cnt.value,
                expanded=expanded.reshape(N, N), input_rows=irows[:prob.num_inputs],
                output_rows=orows[:prob.num_outputs])


def ref_batch_forward(prob: Problem, schema: SchemaSpec, pop_nodes, pop_conns, X, nthreads=1):
    P = pop_nodes.shape[0]
    B = X.shape[0]
    out = np.zeros((P, B, prob.num_outputs))
    bad = C.c_int(-1)
    msg = C.create_string_buffer(512)
    sh, sc = prob.c(), schema.c()
    pop_nodes = np.ascontiguousarray(pop_nodes, dtype=np.float64)
    pop_conns = np.ascontiguousarray(pop_conns, dtype=np.float64)
    X = np.ascontiguousarray(X, dtype=np.float64)
    st = ref().fr_batch_forward(C.byref(sh), C.byref(sc), P, ptr(pop_nodes, F64P), ptr(pop_conns, F64P),
                                ptr(X, F64P), B, ptr(out, F64P), nthreads, C.byref(bad), msg,
                                C.c_size_t(512))
    return st, bad.value, msg.value.decode(), out


def distance(prob, n1, c1, n2, c2, cd=1.0, ch=0.5, use_ref=False) -> float:
    sh = prob.c()
    cfg = DistCfg(cd, ch)
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (n1, c1, n2, c2)]
    f = ref().fr_distance if use_ref else oracle().fo_distance
    if use_ref:
        f.argtypes = [C.POINTER(Shape), F64P, F64P, F64P, F64P, C.POINTER(DistCfg)]
    else:
        f.argtypes = [C.POINTER(Shape), F64P, F64P, F64P, F64P, C.POINTER(DistCfg)]
    return f(C.byref(sh), *[ptr(a, F64P) for a in arrs], C.byref(cfg))


def crossover(prob, fn, fc, on, oc, key: Key, use_ref=False):
    sh = prob.c()
    cn = np.zeros((prob.max_nodes, 5))
    cc = np.zeros((prob.max_conns, 4))
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (fn, fc, on, oc)]
    if use_ref:
        kw = key_words(key)
        ref().fr_crossover(C.byref(sh), *[ptr(a, F64P) for a in arrs], ptr(kw, U32P), ptr(cn, F64P),
                           ptr(cc, F64P))
    else:
        oracle().fo_crossover(C.byref(sh), *[ptr(a, F64P) for a in arrs], key, ptr(cn, F64P),
                              ptr(cc, F64P))
    return cn, cc


def mutate_population(prob, schema, pop_nodes, pop_conns, keys: np.ndarray, cfg: MutCfg,
                      next_key: int, use_ref=False):
    """Sequential mutate of every genome in slot order with one InnovationTable
    (ops.hpp:363-374 composed as in ops.hpp:169-175).  Returns
    (status, bad_genome, next_key, nodes, conns)."""
    sh, sc = prob.c(), schema.c()
    nodes = np.array(pop_nodes, dtype=np.float64, copy=True, order="C")
    conns = np.array(pop_conns, dtype=np.float64, copy=True, order="C")
    P = nodes.shape[0]
    keys = np.ascontiguousarray(keys, dtype=np.uint32).reshape(P, 4)
    if use_ref:
        nk = C.c_int(next_key)
        bad = C.c_int(-1)
        msg = C.create_string_buffer(256)
        st = ref().fr_mutate_population(C.byref(sh), C.byref(sc), P, ptr(nodes, F64P), ptr(conns, F64P),
                                        ptr(keys, U32P), C.byref(cfg), C.byref(nk), C.byref(bad), msg,
                                        C.c_size_t(256))
        return st, bad.value, nk.value, nodes, conns
    t = InnovTable()
    lib = oracle()
    lib.fo_innov_init(C.byref(t), next_key)
    st, bad = 0, -1
    for p in range(P):
        st = lib.fo_mutate(C.byref(sh), C.byref(sc), ptr(nodes[p], F64P), ptr(conns[p], F64P),
                           key_from_words(keys[p]), C.byref(cfg), C.byref(t))
        if st:
            bad = p
            break
    nk = t.next_key
    lib.fo_innov_free(C.byref(t))
    return st, bad, nk, nodes, conns


# ---------------------------------------------------------------------------
# Evolution restatement driver (oracle/evolution.c)
# ---------------------------------------------------------------------------

def neat_cfg(pop_size, max_species=10, threshold=3.5, species_elitism=2, max_stagnation=15, genome_elitism=2,
             survival=0.2, spawn_rate=0.5, output_activation=0, mutation=None, cd=1.0, ch=0.5) -> NeatCfg:
    return NeatCfg(pop_size, max_species, threshold, species_elitism, max_stagnation, genome_elitism, survival,
                   spawn_rate, output_activation, mutation if mutation is not None else mut_cfg(), DistCfg(cd, ch))


class OracleEvolution:
    """The frozen CPU generation loop: speciate -> stagnation -> spawn -> reproduce."""

    def __init__(self, prob: Problem, schema: SchemaSpec, cfg: NeatCfg, seed: int):
        self.prob, self.schema, self.cfg, self.seed = prob, schema, cfg, seed
        self._sh, self._sc = prob.c(), schema.c()
        lib = oracle()
        lib.fo_species_init.argtypes = [C.POINTER(Species), C.POINTER(Shape), C.c_int]
        lib.fo_speciate.argtypes = [C.POINTER(Shape), C.POINTER(NeatCfg), F64P, F64P, C.POINTER(Species), I32P]
        lib.fo_update_stagnation.argtypes = [C.POINTER(NeatCfg), F64P, C.POINTER(Species), I32P]
        lib.fo_compute_spawn.argtypes = [C.POINTER(NeatCfg), F64P, I32P, C.POINTER(Species)]
        self.species = Species()
        lib.fo_species_init(C.byref(self.species), C.byref(self._sh), cfg.max_species)
        P = cfg.pop_size
        self.nodes, self.conns = prob.empty_pop(P)
        self.innov = InnovTable()
        lib.fo_innov_init(C.byref(self.innov), prob.num_inputs + prob.num_outputs + 1)
        self.generation = 0
        self.species_of = np.zeros(P, dtype=np.int32)

    def init_population(self):
        st = oracle().fo_initialize_population(C.byref(self._sh), C.byref(self._sc), C.byref(self.cfg),
                                               C.c_uint64(self.seed), ptr(self.nodes, F64P), ptr(self.conns, F64P))
        assert st == 0, st

    def step(self, fitness: np.ndarray):
        lib = oracle()
        P = self.cfg.pop_size
        f = np.ascontiguousarray(fitness, dtype=np.float64)
        lib.fo_speciate(C.byref(self._sh), C.byref(self.cfg), ptr(self.nodes, F64P), ptr(self.conns, F64P),
                        C.byref(self.species), ptr(self.species_of, I32P))
        lib.fo_update_stagnation(C.byref(self.cfg), ptr(f, F64P), C.byref(self.species), ptr(self.species_of, I32P))
        lib.fo_compute_spawn(C.byref(self.cfg), ptr(f, F64P), ptr(self.species_of, I32P), C.byref(self.species))
        lib.fo_innov_next_generation(C.byref(self.innov))
        nn, nc = self.prob.empty_pop(P)
        pa = np.zeros(P, dtype=np.int32)
        pb = np.zeros(P, dtype=np.int32)
        st = lib.fo_reproduce(C.byref(self._sh), C.byref(self._sc), C.byref(self.cfg), ptr(self.nodes, F64P),
                              ptr(self.conns, F64P), ptr(f, F64P), ptr(self.species_of, I32P),
                              C.byref(self.species), C.c_uint64(self.seed), self.generation, C.byref(self.innov),
                              ptr(nn, F64P), ptr(nc, F64P), ptr(pa, I32P), ptr(pb, I32P))
        assert st == 0, st
        self.nodes, self.conns = nn, nc
        self.last_parents = (pa, pb)
        self.generation += 1

    def set_population(self, nodes, conns):
        """Load a population; the innovation counter moves above its largest
        key (InnovationTable::reserve_up_to), as fnb_evolver_set_population
        + fnb_evolver_set_next_key do."""
        self.nodes = np.array(nodes, dtype=np.float64, copy=True, order="C")
        self.conns = np.array(conns, dtype=np.float64, copy=True, order="C")
        keys = self.nodes[:, :, 0]
        if np.any(~np.isnan(keys)):
            self.innov.next_key = max(self.innov.next_key, int(np.nanmax(keys)) + 1)

    def species_view(self):
        s = self.species
        k = s.count
        return dict(count=k, ids=np.array([s.id[j] for j in range(k)]), spawn=np.array([s.spawn[j] for j in range(k)]),
                    best=np.array([s.best_fitness[j] for j in range(k)]),
                    stagnation=np.array([s.stagnation[j] for j in range(k)]))


# ---- C4 HyperNEAT (oracle/hyperneat.c: this repo's FP64 definition) ----------

class HyperCfg(C.Structure):
    _fields_ = [("n_obs", C.c_int), ("n_act", C.c_int), ("steps", C.c_int), ("weight_threshold", C.c_double),
                ("max_weight", C.c_double), ("act_cost", C.c_double)]


def hyper_cfg(n_obs=27, n_act=8, steps=1000, threshold=0.2, max_weight=3.0, act_cost=0.01) -> HyperCfg:
    return HyperCfg(n_obs, n_act, steps, threshold, max_weight, act_cost)


def hyper_queries(cfg: HyperCfg) -> np.ndarray:
    q = np.zeros(((cfg.n_obs + 1) * cfg.n_act, 5))
    oracle().fo_hyper_queries(C.byref(cfg), ptr(q, F64P))
    return q


def hyper_weight(cfg: HyperCfg, y: float) -> float:
    lib = oracle()
    lib.fo_hyper_weight.restype = C.c_double
    lib.fo_hyper_weight.argtypes = [C.POINTER(HyperCfg), C.c_double]
    return lib.fo_hyper_weight(C.byref(cfg), y)


def hyper_substrate(cfg: HyperCfg, cppn_out) -> np.ndarray:
    y = np.ascontiguousarray(cppn_out, dtype=np.float64)
    W = np.zeros((cfg.n_act, cfg.n_obs + 1))
    oracle().fo_hyper_substrate(C.byref(cfg), ptr(y, F64P), ptr(W, F64P))
    return W


def hyper_rollout(cfg: HyperCfg, W, A, B, s0) -> float:
    lib = oracle()
    lib.fo_hyper_rollout.restype = C.c_double
    w, a, b, s = (np.ascontiguousarray(x, dtype=np.float64) for x in (W, A, B, s0))
    return lib.fo_hyper_rollout(C.byref(cfg), ptr(w, F64P), ptr(a, F64P), ptr(b, F64P), ptr(s, F64P))


def hyper_cppn_outputs(prob: Problem, schema: SchemaSpec, nodes, conns, cfg: HyperCfg, use_ref: bool = True):
    """[P, Q] CPPN outputs at the substrate queries: the reference's own
    batch_forward (oracle/_ref) when available, else the C restatement."""
    X = hyper_queries(cfg)
    if use_ref and ref_available():
        st, bad, msg, out = ref_batch_forward(prob, schema, nodes, conns, X)
        assert st == 0, msg
        return out[:, :, 0]
    outs = []
    for i in range(nodes.shape[0]):
        net = oracle_transform(prob, schema, nodes[i], conns[i])
        outs.append(oracle_forward(prob, schema, nodes[i], net, X)[:, 0])
    return np.stack(outs)


def explain_invalid(prob: Problem, schema: SchemaSpec, nodes, conns, use_ref: bool = True) -> str:
    """explain_invalid (genome.hpp:364-417): the reference's string, '' if valid."""
    buf = C.create_string_buffer(512)
    sh, sc = prob.c(), schema.c()
    n = np.ascontiguousarray(nodes, dtype=np.float64)
    c = np.ascontiguousarray(conns, dtype=np.float64)
    lib = ref() if use_ref and ref_available() else oracle()
    fn = lib.fr_explain_invalid if lib is not oracle() else lib.fo_explain_invalid
    fn(C.byref(sh), C.byref(sc), ptr(n, F64P), ptr(c, F64P), buf, C.c_size_t(512))
    return buf.value.decode()
