"""Host-side mirror of the reference flatneat API over the CUDA C ABI.

Names and meanings follow /root/reference/proj/include/flatneat/:
AttributeSchema / GenomeLimits / PopulationTensors (genome.hpp), transform /
batch_forward / BatchResult (network.hpp), MutationConfig / DistanceConfig /
InnovationTable semantics (ops.hpp) and Error / Errc (errors.hpp).  Failures
raise FlatneatError carrying the reference's Errc name, its what() string
and the lowest failing genome index (parallel.hpp:69-73).

Two call styles:
  * host arrays (numpy) -- synchronous, mirrors the reference free functions;
  * device tensors (torch.cuda) -- asynchronous on the current stream, used by
    the generation loop and the benchmark.
"""
from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _native as N

ERRC = ["unknown_function", "genome_full", "duplicate_key", "duplicate_conn", "dangling_endpoint",
        "key_not_found", "protected_node", "attr_out_of_range", "shape_mismatch", "corrupt_row",
        "cycle_detected", "non_finite_input", "non_finite_state", "empty_aggregation", "empty_dataset",
        "parse_error", "version_unsupported", "limits_too_small", "config_error", "eval_error"]

ACTIVATIONS = {"identity": 0, "tanh": 1, "sigmoid": 2, "relu": 3, "sin": 4}   # functions.hpp:23-30
AGGREGATIONS = {"sum": 0, "product": 1, "max": 2, "mean": 3}                  # functions.hpp:34-40

FIT_NONE, FIT_NEG_MSE, FIT_OFFSET_SSE = 0, 1, 2
NODE_COLS, CONN_COLS = 5, 4


class FlatneatError(RuntimeError):
    """flatneat::Error (errors.hpp:59-69): code name, what() and genome index."""

    def __init__(self, status: int, what: str, index: int = -1):
        self.code = ERRC[status - 1] if 1 <= status <= len(ERRC) else "unknown"
        self.status = status
        self.index = index
        super().__init__(what or self.code)


@dataclass
class AttributeSchema:
    """genome.hpp:42-85; registry order is significant."""
    activations: Sequence[str] = ("tanh",)
    aggregations: Sequence[str] = ("sum",)
    default_activation: int = 0
    default_aggregation: int = 0

    def to_c(self) -> N.fnb_schema:
        s = N.fnb_schema()
        s.n_act = len(self.activations)
        s.n_agg = len(self.aggregations)
        for i, a in enumerate(self.activations):
            if a not in ACTIVATIONS:
                raise FlatneatError(1, f"unknown_function: activation '{a}' is not built in")
            s.act[i] = ACTIVATIONS[a]
        for i, a in enumerate(self.aggregations):
            if a not in AGGREGATIONS:
                raise FlatneatError(1, f"unknown_function: aggregation '{a}' is not built in")
            s.agg[i] = AGGREGATIONS[a]
        s.default_act = self.default_activation
        s.default_agg = self.default_aggregation
        return s


@dataclass
class GenomeLimits:
    """genome.hpp:87-92"""
    max_nodes: int = 50
    max_conns: int = 100


@dataclass
class PopulationTensors:
    """genome.hpp:315-338: pop_nodes [P, N, 5], pop_conns [P, C, 4], FP64, NaN padded."""
    pop_nodes: np.ndarray
    pop_conns: np.ndarray
    input_keys: Sequence[int]
    output_keys: Sequence[int]

    @property
    def pop_size(self) -> int:
        return int(self.pop_nodes.shape[0])

    @property
    def limits(self) -> GenomeLimits:
        return GenomeLimits(int(self.pop_nodes.shape[1]), int(self.pop_conns.shape[1]))


@dataclass
class AttrMutation:
    """ops.hpp:117-123"""
    init_mean: float = 0.0
    init_std: float = 1.0
    mutate_power: float = 0.5
    mutate_rate: float = 0.7
    replace_rate: float = 0.1

    def to_c(self):
        return N.fnb_attr_mutation(self.init_mean, self.init_std, self.mutate_power, self.mutate_rate,
                                   self.replace_rate)


@dataclass
class MutationConfig:
    """ops.hpp:125-135 (Appendix-A defaults)."""
    node_add: float = 0.2
    node_delete: float = 0.0
    conn_add: float = 0.4
    conn_delete: float = 0.0
    bias: AttrMutation = field(default_factory=lambda: AttrMutation(0.0, 1.0, 0.5, 0.7, 0.1))
    response: AttrMutation = field(default_factory=lambda: AttrMutation(1.0, 0.0, 0.0, 0.0, 0.0))
    weight: AttrMutation = field(default_factory=lambda: AttrMutation(0.0, 1.0, 0.5, 0.8, 0.1))
    activation_replace_rate: float = 0.0
    aggregation_replace_rate: float = 0.0

    def to_c(self):
        return N.fnb_mutation_config(self.node_add, self.node_delete, self.conn_add, self.conn_delete,
                                     self.bias.to_c(), self.response.to_c(), self.weight.to_c(),
                                     self.activation_replace_rate, self.aggregation_replace_rate)


@dataclass
class DistanceConfig:
    """ops.hpp:137-140"""
    compatibility_disjoint: float = 1.0
    compatibility_homologous: float = 0.5

    def to_c(self):
        return N.fnb_distance_config(self.compatibility_disjoint, self.compatibility_homologous)


@dataclass
class BatchResult:
    """network.hpp:281-292: values[P][B][O]."""
    values: np.ndarray

    @property
    def pop_size(self):
        return self.values.shape[0]

    @property
    def batch(self):
        return self.values.shape[1]

    @property
    def outputs(self):
        return self.values.shape[2]

    def at(self, p, b, o):
        return float(self.values[p, b, o])


def _dp(a: np.ndarray):
    return a.ctypes.data_as(N.DP)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _stream_handle(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


class Engine:
    """One CUDA context (fnb_ctx) for a fixed genome shape and schema."""

    def __init__(self, limits: GenomeLimits, input_keys: Sequence[int], output_keys: Sequence[int],
                 schema: AttributeSchema = AttributeSchema(), device: int = 0):
        self.limits = limits
        self.input_keys = list(input_keys)
        self.output_keys = list(output_keys)
        self.schema = schema
        self.device = device
        self._ik = (C.c_int * max(1, len(self.input_keys)))(*self.input_keys)
        self._ok = (C.c_int * max(1, len(self.output_keys)))(*self.output_keys)
        shape = N.fnb_shape(limits.max_nodes, limits.max_conns, len(self.input_keys), len(self.output_keys),
                            self._ik, self._ok)
        self._lib = N.lib()
        h = C.c_void_p()
        st = self._lib.fnb_ctx_create(C.byref(shape), C.byref(schema.to_c()), device, C.byref(h))
        if st:
            raise FlatneatError(st, f"{ERRC[st - 1]}: fnb_ctx_create failed")
        self._h = h
        self._dependents = weakref.WeakSet()  # evolvers on this context: closed first

    def close(self):
        if getattr(self, "_h", None):
            for d in list(getattr(self, "_dependents", ())):
                d.close()
            self._lib.fnb_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- helpers -----------------------------------------------------------
    @property
    def num_inputs(self):
        return len(self.input_keys)

    @property
    def num_outputs(self):
        return len(self.output_keys)

    @property
    def net_bytes(self) -> int:
        return int(self._lib.fnb_net_bytes(self._h))

    @property
    def launch_count(self) -> int:
        return int(self._lib.fnb_launch_count(self._h))

    def _raise(self, st: int):
        if st:
            what = self._lib.fnb_last_error(self._h).decode()
            raise FlatneatError(st, what, int(self._lib.fnb_last_error_index(self._h)))

    def _check_pop(self, pop_nodes, pop_conns):
        n, c = _f64(pop_nodes), _f64(pop_conns)
        P = n.shape[0]
        if n.shape != (P, self.limits.max_nodes, NODE_COLS) or c.shape != (P, self.limits.max_conns, CONN_COLS):
            raise FlatneatError(9, "shape_mismatch: population tensors do not match the engine limits")
        return n, c, P

    # -- host layer (network.hpp) -----------------------------------------------
    def transform(self, pop_nodes, pop_conns):
        """transform() of every genome (network.hpp:122-220) -> (order[P,N] int32 with -1 tail, order_count[P])."""
        n, c, P = self._check_pop(pop_nodes, pop_conns)
        order = np.empty((P, self.limits.max_nodes), dtype=np.int32)
        cnt = np.empty(P, dtype=np.int32)
        self._raise(self._lib.fnb_transform(self._h, _dp(n), _dp(c), P, order.ctypes.data_as(N.IP),
                                            cnt.ctypes.data_as(N.IP)))
        return order, cnt

    def batch_forward(self, pop_nodes, pop_conns, inputs, batch: Optional[int] = None) -> BatchResult:
        """transform() + batch_forward() (network.hpp:294-330); FP32 on the device."""
        n, c, P = self._check_pop(pop_nodes, pop_conns)
        x = _f64(inputs).reshape(-1)
        B = batch if batch is not None else x.size // max(1, self.num_inputs)
        if x.size != B * self.num_inputs:
            raise FlatneatError(9, "shape_mismatch: input matrix is not batch x num_inputs")
        out = np.empty((P, B, self.num_outputs), dtype=np.float64)
        self._raise(self._lib.fnb_batch_forward(self._h, _dp(n), _dp(c), P, _dp(x), B, _dp(out)))
        return BatchResult(out)

    def evaluate(self, pop_nodes, pop_conns, inputs, targets, kind: int = FIT_NEG_MSE,
                 offset: float = 0.0) -> np.ndarray:
        """transform + forward + fused fitness -> fitness[P] (FP64)."""
        n, c, P = self._check_pop(pop_nodes, pop_conns)
        x = _f64(inputs).reshape(-1)
        y = _f64(targets).reshape(-1)
        B = x.size // max(1, self.num_inputs)
        if x.size != B * self.num_inputs or y.size != B * self.num_outputs:
            raise FlatneatError(9, "shape_mismatch: inputs/targets are not batch x I / batch x O")
        fit = np.empty(P, dtype=np.float64)
        self._raise(self._lib.fnb_evaluate(self._h, _dp(n), _dp(c), P, _dp(x), _dp(y), B, kind, offset, _dp(fit)))
        return fit

    # -- device layer (torch tensors, current stream) -----------------------------
    def alloc_nets(self, P: int):
        import torch
        return torch.empty(P * self.net_bytes, dtype=torch.uint8, device=f"cuda:{self.device}")

    def transform_d(self, nodes, conns, nets=None, stream=None):
        P = nodes.shape[0]
        if nets is None:
            nets = self.alloc_nets(P)
        self._raise(self._lib.fnb_transform_d(self._h, nodes.data_ptr(), conns.data_ptr(), P, nets.data_ptr(),
                                              _stream_handle(stream)))
        return nets

    def check_nets_d(self, nodes, conns, nets, stream=None):
        self._raise(self._lib.fnb_check_nets_d(self._h, nodes.data_ptr(), conns.data_ptr(), nets.data_ptr(),
                                               nodes.shape[0], _stream_handle(stream)))

    def net_order_d(self, nets, P, stream=None):
        import torch
        order = torch.empty((P, self.limits.max_nodes), dtype=torch.int32, device=nets.device)
        cnt = torch.empty(P, dtype=torch.int32, device=nets.device)
        self._raise(self._lib.fnb_net_order_d(self._h, nets.data_ptr(), P, order.data_ptr(), cnt.data_ptr(),
                                              _stream_handle(stream)))
        return order, cnt

    def forward_d(self, nets, P: int, X, Y=None, kind: int = FIT_NONE, offset: float = 0.0, fitness=None,
                  out=None, stream=None):
        B = X.shape[0]
        self._raise(self._lib.fnb_forward_d(self._h, nets.data_ptr(), P, X.data_ptr(),
                                            Y.data_ptr() if Y is not None else None, B, kind, offset,
                                            fitness.data_ptr() if fitness is not None else None,
                                            out.data_ptr() if out is not None else None, _stream_handle(stream)))
        return fitness if fitness is not None else out


# ---------------------------------------------------------------------------
# RngKey tree (rng.hpp:44-72) -- host helpers over the C ABI
# ---------------------------------------------------------------------------

def key_seed(seed: int) -> np.ndarray:
    """RngKey(seed).words() (rng.hpp:48-56)."""
    out = np.zeros(4, dtype=np.uint32)
    N.lib().fnb_key_seed(C.c_uint64(seed), out.ctypes.data_as(N.U32P))
    return out


def key_split(key, index: int) -> np.ndarray:
    """RngKey::split(index).words() (rng.hpp:58-66)."""
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    N.lib().fnb_key_split(k.ctypes.data_as(N.U32P), C.c_uint64(index), out.ctypes.data_as(N.U32P))
    return out


def _engine_distance(self, pop_nodes, pop_conns, rep_nodes, rep_conns, cfg: DistanceConfig = DistanceConfig()):
    """distance(genome_p, rep_s) (ops.hpp:415-473) -> [P, S], FP64 bit-exact."""
    n, c, P = self._check_pop(pop_nodes, pop_conns)
    rn, rc, S = self._check_pop(rep_nodes, rep_conns)
    out = np.empty((P, S), dtype=np.float64)
    cc = cfg.to_c()
    self._raise(self._lib.fnb_distance(self._h, _dp(n), _dp(c), P, _dp(rn), _dp(rc), S, C.byref(cc), _dp(out)))
    return out


def _engine_crossover(self, fit_nodes, fit_conns, other_nodes, other_conns, keys):
    """crossover(fit, other, key) (ops.hpp:382-407) for n pairs; keys [n, 4] uint32."""
    fn, fc, n = self._check_pop(fit_nodes, fit_conns)
    on, oc, n2 = self._check_pop(other_nodes, other_conns)
    if n2 != n:
        raise FlatneatError(9, "shape_mismatch: parents have different counts")
    k = np.ascontiguousarray(keys, dtype=np.uint32).reshape(n, 4)
    cn = np.empty_like(fn)
    cc = np.empty_like(fc)
    self._raise(self._lib.fnb_crossover(self._h, _dp(fn), _dp(fc), _dp(on), _dp(oc), n, k.ctypes.data_as(N.U32P),
                                        _dp(cn), _dp(cc)))
    return cn, cc


def _engine_distance_d(self, nodes, conns, rep_nodes, rep_conns, out=None, cfg: DistanceConfig = DistanceConfig(),
                       stream=None):
    import torch
    P, S = nodes.shape[0], rep_nodes.shape[0]
    if out is None:
        out = torch.empty((P, S), dtype=torch.float64, device=nodes.device)
    cc = cfg.to_c()
    self._raise(self._lib.fnb_distance_d(self._h, nodes.data_ptr(), conns.data_ptr(), P, rep_nodes.data_ptr(),
                                         rep_conns.data_ptr(), S, C.byref(cc), out.data_ptr(), _stream_handle(stream)))
    return out


def _engine_crossover_d(self, nodes, conns, fit_idx, other_idx, keys, child_nodes, child_conns, stream=None):
    n = fit_idx.shape[0]
    self._raise(self._lib.fnb_crossover_d(self._h, nodes.data_ptr(), conns.data_ptr(), fit_idx.data_ptr(),
                                          other_idx.data_ptr(), keys.data_ptr(), n, child_nodes.data_ptr(),
                                          child_conns.data_ptr(), _stream_handle(stream)))
    return child_nodes, child_conns


def _engine_stream_draws_d(self, keys, n_draws: int, kind: int = 0, n: int = 0, stream=None):
    import torch
    nk = keys.shape[0]
    out = torch.empty((nk, n_draws), dtype=torch.int64, device=keys.device)
    self._raise(self._lib.fnb_stream_draws_d(self._h, keys.data_ptr(), nk, n_draws, kind, C.c_uint64(n),
                                             out.data_ptr(), _stream_handle(stream)))
    return out


def _engine_split_keys_d(self, key, base: int, n: int, out=None, stream=None):
    import torch
    if out is None:
        out = torch.empty((n, 4), dtype=torch.int32, device=f"cuda:{self.device}")
    k = np.ascontiguousarray(key, dtype=np.uint32)
    self._raise(self._lib.fnb_split_keys_d(self._h, k.ctypes.data_as(N.U32P), C.c_uint64(base), n, out.data_ptr(),
                                           _stream_handle(stream)))
    return out


Engine.distance = _engine_distance
Engine.crossover = _engine_crossover
Engine.distance_d = _engine_distance_d
Engine.crossover_d = _engine_crossover_d
Engine.stream_draws_d = _engine_stream_draws_d
Engine.split_keys_d = _engine_split_keys_d


class InnovationTable:
    """The reference's InnovationTable (ops.hpp:145-167): (in, out) -> key memo
    for one generation and a counter that never runs backwards."""

    def __init__(self, first_key: int = 0):
        self._next = int(first_key)
        self._assignments = {}

    def get_or_assign(self, in_key: int, out_key: int) -> int:
        pair = (int(in_key), int(out_key))
        k = self._assignments.get(pair)
        if k is None:
            k = self._next
            self._next += 1
            self._assignments[pair] = k
        return k

    def next_generation(self):
        self._assignments.clear()

    def next_key(self) -> int:
        return self._next

    def reserve_up_to(self, key: int):
        self._next = max(self._next, int(key))


def _engine_mutate(self, pop_nodes, pop_conns, keys, cfg: MutationConfig = MutationConfig(), next_key: int = 0,
                   table: Optional[InnovationTable] = None):
    """mutate() of every genome in slot order (ops.hpp:363-374, 169-175) ->
    (nodes, conns, next_key).  With `table` (an InnovationTable), its
    get_or_assign is called once per splitting slot in slot order, as the
    sequential loop calls it (fnb_mutate_table); without it a fresh
    InnovationTable(next_key) is used on the device.  Raises FlatneatError at
    the lowest failing genome (its .index)."""
    n = np.array(pop_nodes, dtype=np.float64, copy=True, order="C")
    c = np.array(pop_conns, dtype=np.float64, copy=True, order="C")
    P = n.shape[0]
    self._check_pop(n, c)
    k = np.ascontiguousarray(keys, dtype=np.uint32)
    if k.size != 4 * P:
        raise FlatneatError(9, "shape_mismatch: mutate needs one key per genome")
    k = k.reshape(P, 4)
    mc = cfg.to_c()
    if table is not None:
        cb = N.INNOVATION_FN(lambda _u, a, b: table.get_or_assign(a, b))
        st = self._lib.fnb_mutate_table(self._h, _dp(n), _dp(c), P, k.ctypes.data_as(N.U32P), C.byref(mc), cb,
                                        None, None)
        if st:
            err = FlatneatError(st, self._lib.fnb_last_error(self._h).decode(),
                                int(self._lib.fnb_last_error_index(self._h)))
            err.partial = (n, c, table.next_key())
            raise err
        return n, c, table.next_key()
    nk = C.c_int(next_key)
    st = self._lib.fnb_mutate(self._h, _dp(n), _dp(c), P, k.ctypes.data_as(N.U32P), C.byref(mc), C.byref(nk))
    if st:
        err = FlatneatError(st, self._lib.fnb_last_error(self._h).decode(), int(self._lib.fnb_last_error_index(self._h)))
        err.partial = (n, c, nk.value)
        raise err
    return n, c, nk.value


def _engine_mutate_d(self, nodes, conns, keys, next_key, status, cfg: MutationConfig = MutationConfig(),
                     active=None, new_key=None, stream=None):
    P = nodes.shape[0]
    mc = cfg.to_c()
    self._raise(self._lib.fnb_mutate_d(self._h, nodes.data_ptr(), conns.data_ptr(), P, keys.data_ptr(),
                                       active.data_ptr() if active is not None else None, C.byref(mc),
                                       next_key.data_ptr(), status.data_ptr(),
                                       new_key.data_ptr() if new_key is not None else None, _stream_handle(stream)))


Engine.mutate = _engine_mutate
Engine.mutate_d = _engine_mutate_d


# ---- BASELINE config 4: HyperNEAT (include/flatneat_b200.h) ----

@dataclass
class HyperConfig:
    """Substrate and rollout of config 4: num_obs inputs (+ a bias input),
    num_act outputs, `steps` steps of s' = A s + B a with a = tanh(W [s, 1])."""
    num_obs: int = 27
    num_act: int = 8
    steps: int = 1000
    weight_threshold: float = 0.2
    max_weight: float = 3.0
    act_cost: float = 0.01

    def to_c(self) -> N.fnb_hyper_config:
        return N.fnb_hyper_config(self.num_obs, self.num_act, self.steps, self.weight_threshold, self.max_weight,
                                  self.act_cost)


def _engine_hyper_evaluate(self, pop_nodes, pop_conns, cfg: HyperConfig, A, B, s0, weights: bool = False):
    """Fitness of every CPPN genome as a HyperNEAT policy on the linear-dynamics
    rollout -> fitness [P] (and the policy weights [P, num_act, num_obs + 1])."""
    n, c, P = self._check_pop(pop_nodes, pop_conns)
    a = np.ascontiguousarray(A, dtype=np.float64).reshape(cfg.num_obs, cfg.num_obs)
    b = np.ascontiguousarray(B, dtype=np.float64).reshape(cfg.num_obs, cfg.num_act)
    s = np.ascontiguousarray(s0, dtype=np.float64).reshape(cfg.num_obs)
    fit = np.empty(P, dtype=np.float64)
    w = np.empty((P, cfg.num_act, cfg.num_obs + 1), dtype=np.float32) if weights else None
    hc = cfg.to_c()
    self._raise(self._lib.fnb_hyper_evaluate(self._h, _dp(n), _dp(c), P, C.byref(hc), _dp(a), _dp(b), _dp(s),
                                             _dp(fit), w.ctypes.data_as(C.POINTER(C.c_float)) if weights else None))
    return (fit, w) if weights else fit


def _engine_hyper_evaluate_d(self, nets, P: int, cfg: HyperConfig, A, B, s0, fitness, weights=None, stream=None):
    """Device layer: transformed CPPNs `nets` (transform_d), FP32 device A, B, s0;
    FP64 `fitness` [P] (and FP32 `weights`) written on `stream`."""
    hc = cfg.to_c()
    self._raise(self._lib.fnb_hyper_evaluate_d(self._h, nets.data_ptr(), P, C.byref(hc), A.data_ptr(), B.data_ptr(),
                                               s0.data_ptr(), fitness.data_ptr(),
                                               weights.data_ptr() if weights is not None else None,
                                               _stream_handle(stream)))
    return fitness


Engine.hyper_evaluate = _engine_hyper_evaluate
Engine.hyper_evaluate_d = _engine_hyper_evaluate_d


# ---- explain_invalid (genome.hpp:364-417) ------------------------------------------

def explain_message(code: int, detail: int) -> str:
    """The reference's explain_invalid string for a device check code."""
    buf = C.create_string_buffer(128)
    N.lib().fnb_explain_message(int(code), int(detail), buf, 128)
    return buf.value.decode()


def _engine_explain_invalid(self, pop_nodes, pop_conns):
    """explain_invalid of every genome -> list of strings ('' = valid)."""
    n, c, P = self._check_pop(pop_nodes, pop_conns)
    codes = np.empty(P, dtype=np.int32)
    details = np.empty(P, dtype=np.int32)
    self._raise(self._lib.fnb_explain_invalid(self._h, _dp(n), _dp(c), P, codes.ctypes.data_as(N.IP),
                                              details.ctypes.data_as(N.IP)))
    return [explain_message(k, d) if k else "" for k, d in zip(codes, details)]


def _engine_explain_invalid_d(self, nodes, conns, codes, details, stream=None):
    """Device layer: int32 `codes` / `details` [P] for device populations."""
    self._raise(self._lib.fnb_explain_invalid_d(self._h, nodes.data_ptr(), conns.data_ptr(), nodes.shape[0],
                                                codes.data_ptr(), details.data_ptr(), _stream_handle(stream)))


Engine.explain_invalid = _engine_explain_invalid
Engine.explain_invalid_d = _engine_explain_invalid_d
