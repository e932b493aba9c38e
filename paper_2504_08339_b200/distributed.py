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
    collective's stream."""

    def __init__(self, backend, group: Optional[dist.ProcessGroup] = None):
        self.backend = backend
        self.group = group
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
        self.backend.step()
        return fit

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

    def checksum(self) -> int:
        return self.ev.checksum()
