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

    def checksum(self) -> int:
        return self.ev.checksum()
