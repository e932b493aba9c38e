"""Multi-rank generation loop (paper_2504_08339_b200/distributed.py) on CPU.

The sharding and exchange logic -- shard bounds, padded all-gather back into
population order, the fitness injection and the replicated step -- is driven
over gloo at world size 2 with a CPU backend built on the oracle (transform
+ forward per genome, oracle/evolution.c for the step).  Checked: every rank
evaluates only its own shard, the gathered fitness equals a 1-process run's,
and after several generations both ranks hold populations identical to the
1-process run (so the device loop, which runs the same orchestration with
partition-invariant fitness, reproduces the 1-GPU run on N GPUs).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_lib as ol
from paper_2504_08339_b200.distributed import ShardedGeneration, shard_bounds


def host_checksum(nodes: np.ndarray, conns: np.ndarray) -> int:
    """fnb_evolver_checksum's population part, restated on the host."""
    w = np.concatenate([np.ascontiguousarray(nodes).view(np.uint64).ravel(),
                        np.ascontiguousarray(conns).view(np.uint64).ravel()])
    mult = (2 * np.arange(w.size, dtype=np.uint64) + np.uint64(1))
    with np.errstate(over="ignore"):
        return int(np.sum(w * mult, dtype=np.uint64))


class OracleShardBackend:
    """CPU stand-in for DeviceShardBackend: oracle transform + forward for
    fitness (-MSE), OracleEvolution for the step."""

    def __init__(self, P, seed=11):
        self.prob = ol.Problem(16, 40, [0, 1, 2], [3])
        self.schema = ol.SchemaSpec(["tanh", "sigmoid"], ["sum"])
        cfg = ol.neat_cfg(P, max_species=6, threshold=1.0, output_activation=1,
                          mutation=ol.mut_cfg(node_add=0.4, conn_add=0.6))
        self.orc = ol.OracleEvolution(self.prob, self.schema, cfg, seed=seed)
        self.orc.init_population()
        self.pop_size = P
        rng = np.random.default_rng(3)
        self.X = rng.uniform(-1, 1, size=(8, 3))
        self.Y = np.tanh(self.X.sum(axis=1, keepdims=True))
        self.evaluated = []
        self.fitness = None

    def alloc(self, n):
        return torch.zeros(n, dtype=torch.float64)

    def evaluate_range(self, lo, hi, out):
        for i, g in enumerate(range(lo, hi)):
            net = ol.oracle_transform(self.prob, self.schema, self.orc.nodes[g], self.orc.conns[g])
            assert net["status"] == 0
            y = ol.oracle_forward(self.prob, self.schema, self.orc.nodes[g], net, self.X)
            out[i] = -float(np.mean((self.Y - y) ** 2))
        self.evaluated.extend(range(lo, hi))

    def before_collective(self):
        pass

    def after_collective(self):
        pass

    def set_fitness(self, full):
        self.fitness = full[:self.pop_size].numpy().copy()

    def step(self):
        self.orc.step(self.fitness)

    # sharded reproduction: the oracle computes every child; step_back copies
    # only this rank's slots into the next buffers (the rest stay NaN until
    # the all-gather fills them)
    def step_front(self):
        self.orc.step(self.fitness)
        self.staged = (self.orc.nodes.copy(), self.orc.conns.copy())
        self.next = (torch.full(self.staged[0].shape, float("nan"), dtype=torch.float64),
                     torch.full(self.staged[1].shape, float("nan"), dtype=torch.float64))

    def step_back(self, lo, hi):
        self.next[0][lo:hi] = torch.from_numpy(self.staged[0][lo:hi])
        self.next[1][lo:hi] = torch.from_numpy(self.staged[1][lo:hi])
        self.produced = getattr(self, "produced", []) + [(lo, hi)]

    def next_population(self):
        return self.next

    def step_commit(self):
        self.orc.nodes = self.next[0].numpy().copy()
        self.orc.conns = self.next[1].numpy().copy()

    def first_bad(self):
        # the oracle's children never fail: each rank reports "none"
        self.bad = torch.tensor([2 ** 31 - 1], dtype=torch.int32)
        return self.bad

    def checksum(self):
        return host_checksum(self.orc.nodes, self.orc.conns)


def _run(world, rank, P, G, port, outdir, shard_step=False):
    if world > 1:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
    be = OracleShardBackend(P)
    sg = ShardedGeneration(be, shard_step=shard_step)
    fits = []
    for _ in range(G):
        fits.append(sg.generation()[:P].numpy().copy())
    agree = sg.replicas_agree()
    np.savez(os.path.join(outdir, f"w{world}_r{rank}.npz"), fits=np.array(fits), nodes=be.orc.nodes,
             conns=be.orc.conns, evaluated=np.array(be.evaluated), agree=agree, next_key=be.orc.innov.next_key,
             produced=np.array(getattr(be, "produced", [])))
    if world > 1:
        dist.destroy_process_group()


def _worker(rank, world, P, G, port, outdir, shard_step=False):
    _run(world, rank, P, G, port, outdir, shard_step)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("P,world", [(10, 3), (25, 2), (7, 7), (5, 8)])
def test_shard_bounds_cover(P, world):
    b = [shard_bounds(P, world, r) for r in range(world)]
    assert b[0][0] == 0 and b[-1][1] == P
    for (lo, hi), (lo2, _) in zip(b, b[1:]):
        assert hi == lo2
    sizes = [hi - lo for lo, hi in b]
    assert max(sizes) - min(sizes) <= 1


def test_shard_bounds_rejects_bad_rank():
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


@pytest.mark.parametrize("P,shard_step", [(24, False), (25, False), (24, True), (25, True)])
def test_sharded_generations_match_single_process(tmp_path, P, shard_step):
    """Even split and the padded gather; replicated step and sharded reproduction."""
    G = 3
    _run(1, 0, P, G, 0, str(tmp_path))
    mp.spawn(_worker, args=(2, P, G, _free_port(), str(tmp_path), shard_step), nprocs=2, join=True)
    one = np.load(tmp_path / "w1_r0.npz")
    for r in range(2):
        d = np.load(tmp_path / f"w2_r{r}.npz")
        lo, hi = shard_bounds(P, 2, r)
        # each rank evaluated only its shard, every generation
        assert list(d["evaluated"]) == list(range(lo, hi)) * G
        np.testing.assert_array_equal(d["fits"], one["fits"])
        np.testing.assert_array_equal(d["nodes"], one["nodes"])
        np.testing.assert_array_equal(d["conns"], one["conns"])
        assert int(d["next_key"]) == int(one["next_key"])
        assert bool(d["agree"])
        if shard_step:  # each rank produced only its own children, every generation
            assert [tuple(x) for x in d["produced"]] == [(lo, hi)] * G


def test_host_checksum_sensitive():
    be = OracleShardBackend(6)
    h = be.checksum()
    be.orc.conns[3, 0, 3] += 1e-12 if not np.isnan(be.orc.conns[3, 0, 3]) else 0
    be.orc.nodes[0, 0, 1] = 0.125 if be.orc.nodes[0, 0, 1] != 0.125 else 0.25
    assert be.checksum() != h
