"""The generation loop (SPEC.md:328-424 `evolution`; PAPER Algorithm 1) on the device.

NeatConfig mirrors SPEC's NeatConfig with the paper's Appendix C defaults
(PAPER.md:1030-1060).  Evolver wraps fnb_evolver_* (include/flatneat_b200.h):
the population, species state, fitness and innovation counter all stay in
HBM; each `step()` runs speciate -> update_stagnation -> compute_spawn_counts
-> reproduce as device kernels.  `evolve()` is SPEC's evolve(problem, cfg,
key): evaluate, stop at the fitness target BEFORE reproducing, step.
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

from . import _native as N
from .api import (FIT_NEG_MSE, AttributeSchema, DistanceConfig, Engine, FlatneatError, GenomeLimits,
                  MutationConfig, _dp)


@dataclass
class NeatConfig:
    """SPEC.md:333-336 with Appendix C defaults."""
    pop_size: int = 1000
    max_species: int = 10
    compatibility_threshold: float = 3.5
    species_elitism: int = 2
    max_stagnation: int = 15
    genome_elitism: int = 2
    survival_threshold: float = 0.2
    spawn_number_change_rate: float = 0.5
    output_activation: int = 0
    mutation: MutationConfig = field(default_factory=MutationConfig)
    distance: DistanceConfig = field(default_factory=DistanceConfig)
    fitness_target: float = float("inf")
    generation_limit: int = 100

    def to_c(self) -> N.fnb_neat_config:
        return N.fnb_neat_config(self.pop_size, self.max_species, self.compatibility_threshold, self.species_elitism,
                                 self.max_stagnation, self.genome_elitism, self.survival_threshold,
                                 self.spawn_number_change_rate, self.output_activation, self.mutation.to_c(),
                                 self.distance.to_c())


@dataclass
class RunStats:
    """one record per completed generation."""
    generation: int
    best: float
    mean: float
    std: float
    species_count: int
    elapsed_ms: float
    best_index: int = -1
    species_sizes: tuple = ()

    @staticmethod
    def from_c(rs) -> "RunStats":
        k = rs.species_count
        return RunStats(rs.generation, rs.best, rs.mean, rs.std, k, rs.elapsed_ms, rs.best_index,
                        tuple(rs.species_size[j] for j in range(k)))


class Evolver:
    def __init__(self, engine: Engine, cfg: NeatConfig, seed: int):
        self.engine = engine
        self.cfg = cfg
        self.seed = seed
        self._lib = N.lib()
        h = C.c_void_p()
        c = cfg.to_c()
        st = self._lib.fnb_evolver_create(engine._h, C.byref(c), C.c_uint64(seed), C.byref(h))
        if st:
            raise FlatneatError(st, self._lib.fnb_last_error(engine._h).decode())
        self._h = h
        engine._dependents.add(self)

    def close(self):
        # an evolver lives on its engine's context: never destroy it after the context
        if getattr(self, "_h", None) and getattr(self.engine, "_h", None):
            self._lib.fnb_evolver_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _raise(self, st):
        if st:
            raise FlatneatError(st, self._lib.fnb_last_error(self.engine._h).decode(),
                                int(self._lib.fnb_last_error_index(self.engine._h)))

    # -- population ------------------------------------------------------------
    def init_population(self):
        self._raise(self._lib.fnb_evolver_init_population(self._h))

    def population(self):
        P, L = self.cfg.pop_size, self.engine.limits
        n = np.empty((P, L.max_nodes, 5))
        c = np.empty((P, L.max_conns, 4))
        self._raise(self._lib.fnb_evolver_get_population(self._h, _dp(n), _dp(c)))
        return n, c

    def set_population(self, nodes, conns):
        """Load a population; the innovation counter moves above its largest key."""
        n = np.ascontiguousarray(nodes, dtype=np.float64)
        c = np.ascontiguousarray(conns, dtype=np.float64)
        self._raise(self._lib.fnb_evolver_set_population(self._h, _dp(n), _dp(c)))
        keys = n[:, :, 0]
        top = int(np.nanmax(keys)) + 1 if np.any(~np.isnan(keys)) else 0
        self._raise(self._lib.fnb_evolver_set_next_key(self._h, max(top, self.state()[1])))

    def set_population_d(self, nodes, conns):
        """Load a device-resident population (torch float64 tensors on this
        evolver's GPU, pop_size x limits); the innovation counter moves above
        its largest key."""
        import torch
        P, L = self.cfg.pop_size, self.engine.limits
        if tuple(nodes.shape) != (P, L.max_nodes, 5) or tuple(conns.shape) != (P, L.max_conns, 4) \
                or nodes.dtype != torch.float64 or conns.dtype != torch.float64:
            raise ValueError("population must be float64 tensors [pop_size, max_nodes, 5] / [pop_size, max_conns, 4]")
        n, c = nodes.contiguous(), conns.contiguous()
        self._raise(self._lib.fnb_evolver_set_population(self._h, C.cast(n.data_ptr(), N.DP), C.cast(c.data_ptr(), N.DP)))
        keys = n[:, :, 0]
        finite = keys[~torch.isnan(keys)]
        top = int(finite.max().item()) + 1 if finite.numel() else 0
        self._raise(self._lib.fnb_evolver_set_next_key(self._h, max(top, self.state()[1])))

    # -- fitness ----------------------------------------------------------------
    def evaluate(self, X, Y, kind: int = FIT_NEG_MSE, offset: float = 0.0):
        x = np.ascontiguousarray(X, dtype=np.float64)
        y = np.ascontiguousarray(Y, dtype=np.float64)
        self._raise(self._lib.fnb_evolver_evaluate(self._h, _dp(x), _dp(y), x.shape[0], kind, offset))

    def evaluate_d(self, X, Y, kind: int = FIT_NEG_MSE, offset: float = 0.0):
        self._raise(self._lib.fnb_evolver_evaluate_d(self._h, X.data_ptr(), Y.data_ptr(), X.shape[0], kind, offset))

    def eval_check(self):
        """Synchronise and raise the last (device-input) evaluation's error:
        the lowest failing genome's transform error, else non_finite_input
        (fnb_evolver_eval_check)."""
        self._raise(self._lib.fnb_evolver_eval_check(self._h))

    def evaluate_range_d(self, lo: int, hi: int, X, Y, out, kind: int = FIT_NEG_MSE, offset: float = 0.0):
        """Fitness of genomes [lo, hi) into the device FP64 tensor `out` (hi-lo),
        on the evolver stream -- one rank's shard in the multi-GPU loop."""
        if out.numel() < hi - lo or out.dtype != torch_float64():
            raise ValueError("out must be a float64 device tensor of at least hi-lo elements")
        self._raise(self._lib.fnb_evolver_evaluate_range_d(self._h, lo, hi, X.data_ptr(), Y.data_ptr(), X.shape[0],
                                                           kind, offset, out.data_ptr()))

    def set_fitness_d(self, fitness):
        """Device-to-device copy of a full FP64 fitness vector (pop_size)."""
        if fitness.numel() < self.cfg.pop_size or fitness.dtype != torch_float64():
            raise ValueError("fitness must be a float64 device tensor of pop_size elements")
        self._raise(self._lib.fnb_evolver_set_fitness_d(self._h, fitness.data_ptr()))

    def checksum(self) -> int:
        """Population checksum (include/flatneat_b200.h fnb_evolver_checksum)."""
        h = C.c_uint64(0)
        self._raise(self._lib.fnb_evolver_checksum(self._h, C.byref(h)))
        return h.value

    def stream_handle(self) -> int:
        """The evolver's CUDA stream (cudaStream_t as int) -- every evolver
        kernel runs on it; wrap with torch.cuda.ExternalStream to order torch work."""
        return self.device_state()[3]

    def fitness(self) -> np.ndarray:
        f = np.empty(self.cfg.pop_size)
        self._raise(self._lib.fnb_evolver_get_fitness(self._h, _dp(f)))
        return f

    def set_fitness(self, fitness):
        f = np.ascontiguousarray(fitness, dtype=np.float64)
        self._raise(self._lib.fnb_evolver_set_fitness(self._h, _dp(f)))

    # -- generation ---------------------------------------------------------------
    def step(self):
        self._raise(self._lib.fnb_evolver_step(self._h))

    def validate(self) -> int:
        """explain_invalid over the current population on the device: -1 when
        every genome is valid; else raises FlatneatError (corrupt_row) whose
        message is the reference's explanation and .index the genome."""
        bad = C.c_int(-1)
        self._raise(self._lib.fnb_evolver_validate(self._h, C.byref(bad)))
        return bad.value

    # -- the step split for sharded reproduction (distributed.py) -------------------
    def step_front(self):
        """Speciate, stagnation, spawn, parent selection, split plans and
        innovation keys for all slots (fnb_evolver_step_front)."""
        self._raise(self._lib.fnb_evolver_step_front(self._h))

    def step_back(self, lo: int, hi: int):
        """Children [lo, hi) into the next population buffer."""
        self._raise(self._lib.fnb_evolver_step_back(self._h, lo, hi))

    def step_commit(self):
        """The next buffer becomes the population (after the all-gather)."""
        self._raise(self._lib.fnb_evolver_step_commit(self._h))

    def next_population_d(self):
        """Zero-copy torch views (float64) of the next population buffer:
        nodes [pop_size, max_nodes, 5], conns [pop_size, max_conns, 4]."""
        import torch
        n, c = C.c_void_p(), C.c_void_p()
        self._raise(self._lib.fnb_evolver_next_population(self._h, C.byref(n), C.byref(c)))
        P, L = self.cfg.pop_size, self.engine.limits
        dev = torch.device("cuda", self.engine.device)
        return (torch.as_tensor(_DeviceArray(n.value, (P, L.max_nodes, 5)), device=dev),
                torch.as_tensor(_DeviceArray(c.value, (P, L.max_conns, 4)), device=dev))

    def species(self):
        cnt = C.c_int(0)
        ids = np.zeros(32, dtype=np.int32)
        sizes = np.zeros(32, dtype=np.int32)
        spawn = np.zeros(32, dtype=np.int32)
        best = np.zeros(32)
        stag = np.zeros(32, dtype=np.int32)
        sof = np.zeros(self.cfg.pop_size, dtype=np.int32)
        ip = lambda a: a.ctypes.data_as(N.IP)
        self._raise(self._lib.fnb_evolver_species(self._h, C.byref(cnt), ip(ids), ip(sizes), ip(spawn), _dp(best),
                                                  ip(stag), ip(sof)))
        k = cnt.value
        return dict(count=k, ids=ids[:k], sizes=sizes[:k], spawn=spawn[:k], best=best[:k], stagnation=stag[:k],
                    species_of=sof)

    def state(self):
        g, nk = C.c_int(0), C.c_int(0)
        self._raise(self._lib.fnb_evolver_state(self._h, C.byref(g), C.byref(nk)))
        return g.value, nk.value

    # -- checkpoint / resume (fnb_evolver_get_state / set_state) ------------------------
    def get_state(self):
        """(state dict, representative nodes [S,N,5], representative conns [S,C,4])."""
        st = N.fnb_run_state()
        L = self.engine.limits
        rn = np.empty((32, L.max_nodes, 5))
        rc = np.empty((32, L.max_conns, 4))
        self._raise(self._lib.fnb_evolver_get_state(self._h, C.byref(st), _dp(rn), _dp(rc)))
        k = st.species_count
        d = dict(seed=int(st.seed), generation=st.generation, next_key=st.next_key, next_species_id=st.next_species_id,
                 species_id=[st.species_id[j] for j in range(k)], species_best=[st.species_best[j] for j in range(k)],
                 species_stagnation=[st.species_stagnation[j] for j in range(k)],
                 species_size=[st.species_size[j] for j in range(k)],
                 species_spawn=[st.species_spawn[j] for j in range(k)])
        return d, rn[:k].copy(), rc[:k].copy()

    def set_state(self, state: dict, rep_nodes, rep_conns):
        st = N.fnb_run_state()
        k = len(state["species_id"])
        st.seed, st.generation, st.next_key = state["seed"], state["generation"], state["next_key"]
        st.species_count, st.next_species_id = k, state["next_species_id"]
        for j in range(k):
            st.species_id[j] = state["species_id"][j]
            st.species_best[j] = state["species_best"][j]
            st.species_stagnation[j] = state["species_stagnation"][j]
            st.species_size[j] = state["species_size"][j]
            st.species_spawn[j] = state["species_spawn"][j]
        rn = np.ascontiguousarray(rep_nodes, dtype=np.float64)
        rc = np.ascontiguousarray(rep_conns, dtype=np.float64)
        self._raise(self._lib.fnb_evolver_set_state(self._h, C.byref(st), _dp(rn), _dp(rc)))

    def save_checkpoint(self) -> str:
        """The whole run state as one wire document (wire.save_checkpoint)."""
        from .wire import save_checkpoint
        state, rn, rc = self.get_state()
        n, c = self.population()
        sch = self.engine.schema
        return save_checkpoint(state, rn, rc, n, c, self.engine.input_keys, self.engine.output_keys,
                               sch.activations, sch.aggregations)

    def load_checkpoint(self, text: str):
        """Restore population, species table, innovation counter, generation and
        seed; the run then continues bit for bit."""
        from .wire import load_checkpoint
        state, rn, rc, n, c, meta = load_checkpoint(text)
        L = self.engine.limits
        if n.shape != (self.cfg.pop_size, L.max_nodes, 5) or c.shape != (self.cfg.pop_size, L.max_conns, 4):
            raise FlatneatError(9, "shape_mismatch: checkpoint population does not match this evolver")
        if meta["input_keys"] != list(self.engine.input_keys) or meta["output_keys"] != list(self.engine.output_keys):
            raise FlatneatError(9, "shape_mismatch: checkpoint input/output keys differ")
        pn = np.ascontiguousarray(n)
        pc = np.ascontiguousarray(c)
        self._raise(self._lib.fnb_evolver_set_population(self._h, _dp(pn), _dp(pc)))
        self.set_state(state, rn, rc)

    # -- SPEC evolve on the device (fnb_evolve) -----------------------------------------
    def run(self, X, Y, kind: int = FIT_NEG_MSE, offset: float = 0.0, fitness_target: float = float("inf"),
            generation_limit: int = 100, on_generation: Optional[Callable[[RunStats], None]] = None):
        """fnb_evolve: evaluate -> stop at the target -> step, one CUDA graph per
        generation.  Returns (best (nodes, conns), best fitness, [RunStats])."""
        x = np.ascontiguousarray(X, dtype=np.float64)
        y = np.ascontiguousarray(Y, dtype=np.float64)
        B = x.shape[0] if x.ndim > 1 else x.size // max(1, self.engine.num_inputs)
        stats: List[RunStats] = []

        def cb(_user, p):
            rs = RunStats.from_c(p.contents)
            stats.append(rs)
            if on_generation:
                return 1 if on_generation(rs) else 0
            return 0

        fn = N.RUN_STATS_FN(cb)
        L = self.engine.limits
        bn = np.full((L.max_nodes, 5), np.nan)
        bc = np.full((L.max_conns, 4), np.nan)
        bf = C.c_double(float("nan"))
        gens = C.c_int(0)
        self._raise(self._lib.fnb_evolve(self._h, _dp(x), _dp(y), B, kind, offset, fitness_target, generation_limit,
                                         C.cast(fn, C.c_void_p), None, _dp(bn), _dp(bc), C.byref(bf),
                                         C.byref(gens)))
        return (bn, bc), bf.value, stats

    # -- the step sharded over ranks (fnb_evolver_shard_*, distributed.ShardedEvolution) --
    SHARD_PHASES = ("begin", "min_unassigned", "found", "join", "assign_rest", "rep_argmin", "rep_stage",
                    "rep_commit", "compact", "stagnation", "select", "pack", "back")

    def shard_init(self, bounds):
        """Rank r of len(bounds)-1 owns genomes [bounds[r], bounds[r+1])."""
        b = (C.c_int * len(bounds))(*[int(x) for x in bounds])
        self._raise(self._lib.fnb_evolver_shard_init(self._h, len(bounds) - 1, b))
        self._shard_world = len(bounds) - 1

    def shard_phase(self, name: str, rank: int, a: int = 0, b: int = 0):
        """One phase (include/flatneat_b200.h fnb_shard_phase); "select"
        returns the parents each rank holds (a host list, synchronising)."""
        out = (C.c_int * max(1, self._shard_world))() if name == "select" else None
        self._raise(self._lib.fnb_evolver_shard_phase(self._h, self.SHARD_PHASES.index(name), rank, a, b, out))
        return list(out) if out is not None else None

    def shard_buffers(self, M: int = 0):
        """Zero-copy torch views of the buffers the collectives act on."""
        import torch
        sb = N.fnb_shard_buffers()
        self._raise(self._lib.fnb_evolver_shard_buffers(self._h, C.byref(sb)))
        P, L = self.cfg.pop_size, self.engine.limits
        dev = torch.device("cuda", self.engine.device)
        gn, gc = L.max_nodes * 5, L.max_conns * 4

        def view(ptr, n, typestr):
            return torch.as_tensor(_DeviceArray(ptr, (n,), typestr), device=dev)

        out = dict(min_unassigned=view(sb.min_unassigned, 1, "<i4"), rep_dmin=view(sb.rep_dmin, 32, "<i8"),
                   rep_argmin=view(sb.rep_argmin, 32, "<i4"), rep_stage=view(sb.rep_stage, sb.rep_stage_words, "<i8"),
                   species_size=view(sb.species_size, 32, "<i4"), species_max=view(sb.species_max, 32, "<i8"),
                   rank_sum=view(sb.rank_sum, 32, "<i8"), rank_count=view(sb.rank_count, 32, "<i4"),
                   first_bad=view(sb.first_bad, 1, "<i4"), fitness=view(sb.fitness, P, "<f8"),
                   species_of=view(sb.species_of, P, "<i4"), rep_nodes=view(sb.rep_nodes, 32 * gn, "<f8"),
                   rep_conns=view(sb.rep_conns, 32 * gc, "<f8"))
        if M > 0 and sb.send_nodes:
            W = self._shard_world
            out.update(send_nodes=view(sb.send_nodes, M * gn, "<f8"), send_conns=view(sb.send_conns, M * gc, "<f8"),
                       pool_nodes=view(sb.pool_nodes, W * M * gn, "<f8"),
                       pool_conns=view(sb.pool_conns, W * M * gc, "<f8"))
        return out

    def state_species(self) -> int:
        """Species count before the next step (the library's host mirror, no sync)."""
        return int(self._lib.fnb_evolver_host_species(self._h))

    def run_mode(self) -> int:
        """2: the last run() used one CUDA graph per generation (conditional
        step node); 1: evaluate graph + host check + step graph; 0: eager."""
        return int(self._lib.fnb_evolver_run_mode(self._h))

    def device_state(self):
        n, c, f, s = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
        self._raise(self._lib.fnb_evolver_device_state(self._h, C.byref(n), C.byref(c), C.byref(f), C.byref(s)))
        return n.value, c.value, f.value, s.value


class _DeviceArray:
    """__cuda_array_interface__ for a device buffer owned by the library."""

    def __init__(self, ptr: int, shape, typestr: str = "<f8"):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def torch_float64():
    import torch
    return torch.float64


def evolve(engine: Engine, cfg: NeatConfig, seed: int, X=None, Y=None, kind: int = FIT_NEG_MSE, offset: float = 0.0,
           on_generation: Optional[Callable[[RunStats], None]] = None, fitness_fn=None,
           evolver: Optional[Evolver] = None):
    """SPEC.md:392-400 evolve(problem, cfg, key): evaluate -> stop when
    max(fit) >= fitness_target (BEFORE reproducing) -> speciate / stagnate /
    apportion / reproduce, for at most cfg.generation_limit generations.

    The problem is the func-fit / xor dataset (X, Y, kind, offset), run on the
    device by fnb_evolve (one CUDA graph per generation), or any host-side
    `fitness_fn(nodes, conns) -> fitness[P]` (a user problem; its fitness is
    injected each generation).  `evolver` continues an existing run (e.g. one
    restored from a checkpoint) instead of a fresh initialize_population.
    Returns (pop[argmax(fit)] of the last evaluated generation as (nodes,
    conns), its fitness, [RunStats])."""
    ev = evolver
    if ev is None:
        ev = Evolver(engine, cfg, seed)
        ev.init_population()
    if fitness_fn is None:
        return ev.run(X, Y, kind, offset, cfg.fitness_target, cfg.generation_limit, on_generation)
    stats: List[RunStats] = []
    best = (None, float("nan"))
    for _ in range(cfg.generation_limit):
        t0 = time.perf_counter()
        gen = ev.state()[0]
        n, c = ev.population()
        fit = np.ascontiguousarray(fitness_fn(n, c), dtype=np.float64)
        if fit.shape != (cfg.pop_size,) or not np.all(np.isfinite(fit)):
            raise FlatneatError(1 + 19, f"eval_error: generation {gen}: fitness_fn must return pop_size finite values")
        ev.set_fitness(fit)
        i = int(np.argmax(fit))  # lowest index on ties
        best = ((n[i].copy(), c[i].copy()), float(fit[i]))
        done = fit[i] >= cfg.fitness_target
        if not done:
            ev.step()
        sp = ev.species()
        rs = RunStats(gen, float(fit[i]), float(fit.mean()), float(fit.std()), sp["count"],
                      (time.perf_counter() - t0) * 1e3, i, tuple(int(x) for x in sp["sizes"]))
        stats.append(rs)
        if on_generation and on_generation(rs):
            break
        if done:
            break
    return best[0], best[1], stats
