"""Multi-GPU generation loop (SURVEY.md section 8 row e).

One process per GPU (torch.distributed, NCCL over NVLink).  The reference's
generation step is a pure function of (population, species state, fitness,
RngKey) -- every random decision is a Philox draw keyed by (generation, slot)
(E1 in DESIGN.md) -- so the layout is:

* population, species state and the innovation counter are REPLICATED: every
  rank runs the same device `step()` and ends with a bit-identical population
  (checked with `fnb_evolver_checksum`);
* evaluation -- transform + batched forward + fitness, the dominant cost -- is
  SHARDED by contiguous genome blocks (`shard_bounds`);
* the one real exchange is the fitness vector: each rank's FP64 shard is
  all-gathered (`all_gather_into_tensor`, padded to the largest shard) and
  injected device-to-device before the step.

With `shard_step=True` the reproduction is sharded too (config 5 scale,
where crossover + mutation dominate the step): every rank runs the step's
front -- speciation, stagnation, spawn, parent selection, node-split plans
and innovation keys for ALL slots (cheap, replicated) -- then produces only
its own children [lo, hi) (K5 + K6), and the next population is all-gathered
(`all_gather_into_tensor` of the node and connection rows) before every rank
commits it.  Children are independent given the plans, so the population
stays bit-identical to the replicated step.

Fitness is partition-invariant on the device (forward.cu sums fixed
32-sample units in order), so an N-rank run reproduces the 1-GPU run bit for
bit.  The orchestration here is backend-neutral: `DeviceShardBackend` drives
the CUDA library; tests/ drive the same `ShardedGeneration` with a CPU
backend over gloo (world size 2) to check the sharding and exchange logic.
"""
from __future__ import annotations

from typing import List, Optional, Tuple

import torch
import torch.distributed as dist

from .api import FIT_NEG_MSE


def shard_bounds(pop_size: int, world: int, rank: int) -> Tuple[int, int]:
    """Genomes [lo, hi) evaluated by `rank`: contiguous blocks whose sizes
    differ by at most one (the first pop_size % world ranks take one more)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    base, rem = divmod(pop_size, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


class ShardedGeneration:
    """Evaluate this rank's shard, all-gather the fitness, step the replica.

    `backend` provides: pop_size, alloc(n) -> tensor (FP64, on the backend's
    device), evaluate_range(lo, hi, out), set_fitness(full), step(),
    checksum() -> int, and the stream hooks before_collective() /
    after_collective() that order the backend's work against the
    collective's stream; for `shard_step` also step_front(),
    step_back(lo, hi), next_population() -> (nodes, conns) tensors that alias
    the next population, and step_commit()."""

    def __init__(self, backend, group: Optional[dist.ProcessGroup] = None, shard_step: bool = False):
        self.backend = backend
        self.group = group
        self.shard_step = shard_step
        if dist.is_available() and dist.is_initialized():
            self.world = dist.get_world_size(group)
            self.rank = dist.get_rank(group)
        else:
            self.world, self.rank = 1, 0
        P = backend.pop_size
        self.bounds: List[Tuple[int, int]] = [shard_bounds(P, self.world, r) for r in range(self.world)]
        self.shard = max(hi - lo for lo, hi in self.bounds)
        # persistent buffers: they are used on the backend's stream, so they
        # must not come back through the caching allocator mid-generation
        self.local = backend.alloc(self.shard)
        self.gathered = backend.alloc(self.shard * self.world) if self.world > 1 else None
        self.full = backend.alloc(P) if self.world > 1 and self.shard * self.world != P else None
        if self.full is not None:  # padded gather layout -> population order
            idx = [r * self.shard + i for r, (lo, hi) in enumerate(self.bounds) for i in range(hi - lo)]
            self.unpad = torch.tensor(idx, dtype=torch.long, device=self.local.device)

    def evaluate(self) -> torch.Tensor:
        """Fitness of the whole population (FP64, on every rank)."""
        lo, hi = self.bounds[self.rank]
        self.backend.evaluate_range(lo, hi, self.local)
        if self.world == 1:
            full = self.local
        else:
            self.backend.before_collective()
            dist.all_gather_into_tensor(self.gathered, self.local, group=self.group)
            if self.full is not None:
                torch.index_select(self.gathered, 0, self.unpad, out=self.full)
                full = self.full
            else:
                full = self.gathered
            self.backend.after_collective()
        self.backend.set_fitness(full)
        return full

    def generation(self) -> torch.Tensor:
        fit = self.evaluate()
        if self.world == 1 or not self.shard_step:
            self.backend.step()
        else:
            self.reproduce_sharded()
        return fit

    def _gather_rows(self, t: torch.Tensor):
        """All-gather t's row blocks [lo, hi) of every rank into t itself."""
        lo, hi = self.bounds[self.rank]
        row = t[0].numel()
        local = self._scratch(self.shard * row, t)
        local[:(hi - lo) * row].copy_(t[lo:hi].reshape(-1))
        flat = t.view(-1)
        if self.shard * self.world == t.shape[0]:  # equal shards: gather straight into place
            dist.all_gather_into_tensor(flat, local, group=self.group)
        else:  # padded blocks, then back into population order
            padded = self._scratch(self.shard * self.world * row, t, slot=1)
            dist.all_gather_into_tensor(padded, local, group=self.group)
            for r, (a, b) in enumerate(self.bounds):
                flat[a * row:b * row].copy_(padded[r * self.shard * row:(r * self.shard + b - a) * row])

    def _scratch(self, n: int, like: torch.Tensor, slot: int = 0) -> torch.Tensor:
        key = (slot, n, like.dtype, like.device)
        bufs = self.__dict__.setdefault("_bufs", {})
        if key not in bufs:
            bufs[key] = torch.empty(n, dtype=like.dtype, device=like.device)
        return bufs[key]

    def reproduce_sharded(self):
        """The step with this rank producing only children [lo, hi)."""
        lo, hi = self.bounds[self.rank]
        self.backend.step_front()
        self.backend.step_back(lo, hi)
        nodes, conns = self.backend.next_population()
        self.backend.before_collective()
        self._gather_rows(nodes)
        self._gather_rows(conns)
        # every rank must see the lowest failing child, or a failure on one
        # rank leaves the others waiting in the next collective
        bad = self.backend.first_bad()
        if bad is not None and self.world > 1:
            dist.all_reduce(bad, op=dist.ReduceOp.MIN, group=self.group)
        self.backend.after_collective()
        self.backend.step_commit()

    def replicas_agree(self) -> bool:
        """True when every rank holds the same population (checksum gather)."""
        h = self.backend.checksum()
        if self.world == 1:
            return True
        mine = torch.tensor([h & 0xFFFFFFFF, h >> 32], dtype=torch.int64, device=self.local.device)
        allh = [torch.empty_like(mine) for _ in range(self.world)]
        dist.all_gather(allh, mine, group=self.group)
        return all(torch.equal(a, allh[0]) for a in allh)


class DeviceShardBackend:
    """The CUDA library behind ShardedGeneration: an `Evolver` (whose kernels
    all run on its own stream) plus resident device inputs X [B, I] and
    targets Y [B, O] (FP32)."""

    def __init__(self, evolver, X: torch.Tensor, Y: torch.Tensor, kind: int = FIT_NEG_MSE, offset: float = 0.0):
        if not (X.is_cuda and Y.is_cuda and X.dtype == torch.float32 and Y.dtype == torch.float32):
            raise ValueError("X and Y must be float32 CUDA tensors")
        self.ev = evolver
        self.X, self.Y = X.contiguous(), Y.contiguous()
        self.kind, self.offset = kind, offset
        self.pop_size = evolver.cfg.pop_size
        self.device = X.device
        self.stream = torch.cuda.ExternalStream(evolver.stream_handle(), device=self.device)

    def alloc(self, n: int) -> torch.Tensor:
        return torch.zeros(n, dtype=torch.float64, device=self.device)

    def evaluate_range(self, lo: int, hi: int, out: torch.Tensor):
        self.ev.evaluate_range_d(lo, hi, self.X, self.Y, out, self.kind, self.offset)

    def before_collective(self):  # the collective's stream waits for the shard
        torch.cuda.current_stream(self.device).wait_stream(self.stream)

    def after_collective(self):  # the evolver waits for the gathered vector
        self.stream.wait_stream(torch.cuda.current_stream(self.device))

    def set_fitness(self, full: torch.Tensor):
        self.ev.set_fitness_d(full)

    def step(self):
        self.ev.step()

    def step_front(self):
        self.ev.step_front()

    def step_back(self, lo: int, hi: int):
        self.ev.step_back(lo, hi)

    def next_population(self):
        return self.ev.next_population_d()

    def step_commit(self):
        self.ev.step_commit()

    def first_bad(self):
        """The evolver's lowest-failing-child word (device int32 view)."""
        if not hasattr(self, "_first_bad"):
            self.ev.shard_init([0, self.pop_size])
            self._first_bad = self.ev.shard_buffers()["first_bad"]
        return self._first_bad

    def checksum(self) -> int:
        return self.ev.checksum()


_I64_MIN = -(2 ** 63)


class ShardedEvolution:
    """The whole generation sharded over ranks (north star):
    rank r owns genomes [lo, hi) -- it evaluates them, computes their
    speciation distances and produces children [lo, hi) -- and the ranks
    exchange only what the step reduces:

    * the fitness vector (all-gather of FP64 shards);
    * speciation: per founding round an all-reduce MIN of the lowest
      unassigned genome and a broadcast of the founder from its owner; the
      new representatives as MIN of (distance bits, index) and a SUM of
      bit-staged genomes (zeros off the owner); species sizes (SUM);
    * stagnation: species max fitness (MAX of order-preserving bits);
    * spawn: per-species integer sums of 2 x mid-rank (SUM; ranks come from
      the gathered fitness on every rank);
    * reproduce: species ids (all-gather), then the selected parents
      themselves (all-gather of each rank's parents, padded to the largest
      count) -- children read their parents from that pool;
    * the lowest failing child (MIN), so every rank raises together.

    Every reduction is over integers or bit patterns, so the result equals the
    one-process step bit for bit for any world size (the test runs the device
    backend at world sizes 1 and 2).  Collectives run on the evolver's stream
    (torch.cuda.stream context), NCCL on GPUs, gloo in tests."""

    def __init__(self, evolver, X, Y, kind: int = FIT_NEG_MSE, offset: float = 0.0,
                 group: Optional[dist.ProcessGroup] = None):
        self.ev = evolver
        self.X, self.Y, self.kind, self.offset = X, Y, kind, offset
        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        else:
            self.world, self.rank = 1, 0
        P = evolver.cfg.pop_size
        self.P = P
        self.bounds = [shard_bounds(P, self.world, r)[0] for r in range(self.world)] + [P]
        self.lo, self.hi = self.bounds[self.rank], self.bounds[self.rank + 1]
        self.shard = max(self.bounds[r + 1] - self.bounds[r] for r in range(self.world))
        evolver.shard_init(self.bounds)
        self.buf = evolver.shard_buffers()
        self.device = self.buf["fitness"].device
        self.stream = torch.cuda.ExternalStream(evolver.stream_handle(), device=self.device)
        L = evolver.engine.limits
        self.gn, self.gc = L.max_nodes * 5, L.max_conns * 4
        if self.world > 1:
            pad = self.shard * self.world
            self.g_fit = torch.empty(pad, dtype=torch.float64, device=self.device)
            self.g_sp = torch.empty(pad, dtype=torch.int32, device=self.device)
            idx = [r * self.shard + i for r in range(self.world) for i in range(self.bounds[r + 1] - self.bounds[r])]
            self.unpad = torch.tensor(idx, dtype=torch.long, device=self.device)
            self.l_fit = torch.empty(self.shard, dtype=torch.float64, device=self.device)
            self.l_sp = torch.zeros(self.shard, dtype=torch.int32, device=self.device)
        self.collectives = 0
        self.host_syncs = 0

    # -- collectives (no-ops at world size 1) -------------------------------------------
    def _reduce(self, t, op):
        if self.world > 1:
            dist.all_reduce(t, op=op, group=self.group)
            self.collectives += 1

    def _gather_shard(self, full, local, gathered):
        """full[lo:hi] of every rank -> full (padded all-gather, back in order)."""
        if self.world == 1:
            return
        n = self.hi - self.lo
        local[:n].copy_(full[self.lo:self.hi])
        dist.all_gather_into_tensor(gathered, local, group=self.group)
        torch.index_select(gathered, 0, self.unpad, out=full)
        self.collectives += 1

    def _owner(self, g: int) -> int:
        r = 0
        while r + 1 < self.world and self.bounds[r + 1] <= g:
            r += 1
        return r

    # -- one generation -------------------------------------------------------------------
    def evaluate(self):
        """Fitness of the shard, gathered into the evolver's full vector."""
        ev, b = self.ev, self.buf
        with torch.cuda.stream(self.stream):
            ev.evaluate_range_d(self.lo, self.hi, self.X, self.Y, b["fitness"][self.lo:], self.kind, self.offset)
            self._gather_shard(b["fitness"], getattr(self, "l_fit", None), getattr(self, "g_fit", None))

    def step(self):
        ev, b, r = self.ev, self.buf, self.rank
        MIN, MAX, SUM = dist.ReduceOp.MIN, dist.ReduceOp.MAX, dist.ReduceOp.SUM
        with torch.cuda.stream(self.stream):
            S = ev.state_species()  # species before this step (replicated on every rank)
            ev.shard_phase("begin", r)
            while S < ev.cfg.max_species:  # founding rounds (oracle E2)
                ev.shard_phase("min_unassigned", r)
                self._reduce(b["min_unassigned"], MIN)
                f = int(b["min_unassigned"].item())
                self.host_syncs += 1
                if f == 2 ** 31 - 1:
                    break
                ev.shard_phase("found", r, f, S)
                if self.world > 1:
                    o = self._owner(f)
                    dist.broadcast(b["rep_nodes"][S * self.gn:(S + 1) * self.gn], src=o, group=self.group)
                    dist.broadcast(b["rep_conns"][S * self.gc:(S + 1) * self.gc], src=o, group=self.group)
                    self.collectives += 2
                ev.shard_phase("join", r, 0, S)
                S += 1
            ev.shard_phase("assign_rest", r)
            self._reduce(b["rep_dmin"], MIN)
            ev.shard_phase("rep_argmin", r)
            self._reduce(b["rep_argmin"], MIN)
            ev.shard_phase("rep_stage", r)
            self._reduce(b["rep_stage"], SUM)
            ev.shard_phase("rep_commit", r)
            self._reduce(b["species_size"], SUM)
            ev.shard_phase("compact", r)
            if self.world > 1:  # order-preserving bits compare as signed after flipping the top bit
                m = b["species_max"]
                m.bitwise_xor_(_I64_MIN)
                self._reduce(m, MAX)
                m.bitwise_xor_(_I64_MIN)
            ev.shard_phase("stagnation", r)
            self._reduce(b["rank_sum"], SUM)
            self._reduce(b["rank_count"], SUM)
            self._gather_shard(b["species_of"], getattr(self, "l_sp", None), getattr(self, "g_sp", None))
            counts = ev.shard_phase("select", r)
            self.host_syncs += 1
            M = max(1, max(counts))
            ev.shard_phase("pack", r, M)
            b = self.buf = ev.shard_buffers(M)
            if self.world > 1:
                dist.all_gather_into_tensor(b["pool_nodes"], b["send_nodes"], group=self.group)
                dist.all_gather_into_tensor(b["pool_conns"], b["send_conns"], group=self.group)
                self.collectives += 2
            else:  # one rank: its send buffer is the pool
                b["pool_nodes"].copy_(b["send_nodes"])
                b["pool_conns"].copy_(b["send_conns"])
            ev.shard_phase("back", r, M)
            self._reduce(b["first_bad"], MIN)
            self.parents_exchanged = int(sum(counts))
        ev.step_commit()

    def generation(self):
        self.evaluate()
        self.step()

    def local_population(self):
        """This rank's genomes [lo, hi) (host numpy)."""
        n, c = self.ev.population()
        return n[self.lo:self.hi], c[self.lo:self.hi]
