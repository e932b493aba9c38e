"""Benchmark: network evals/s of the NEAT evaluation step at BASELINE config 2,
and generations/s of the full generation loop.

Headline step = transform (K1) + forward with the fused func-fit fitness (K2)
of the pop-10k population (N_max=64, C_max=256, fill 0.75, tanh/sum) over a
1024-sample batch.  At N GPUs the SAME 10k population is split into N genome
blocks (strong scaling, the metric's "pop 10k"), plus the fitness all-gather
(the real per-generation exchange); a weak-scaled line (10k per GPU) is
reported beside it.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Rank 0 prints one JSON line.  --impl reference times the reference's own CPU
path (oracle/_ref = the unmodified reference headers, all host threads) on
the full workload every step; it loads no part of this repo's CUDA library.
"""
from __future__ import annotations

import argparse
import importlib.util
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "network evals/sec (genomes x inputs) at pop 10k"
UNIT = "evals/s"
POP, N_MAX, C_MAX, FILL, BATCH, NI, NO = 10_000, 64, 256, 0.75, 1024, 4, 1
P_SHARD = POP  # per-GPU population of the weak-scaled line and the single-GPU sections
POP_SEED = 1000
WORKLOAD = "C2 func-regression: pop 10k, B=1024, N_max=64, C_max=256, fill 0.75, tanh/sum"


def synthetic():
    """paper_2504_08339_b200/synthetic.py loaded by path: data generation only,
    without importing the package (whose import loads the CUDA library)."""
    spec = importlib.util.spec_from_file_location("fnb_synthetic",
                                                  os.path.join(ROOT, "paper_2504_08339_b200", "synthetic.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def config_dict(world: int) -> dict:
    """The workload both arms run (identical dicts)."""
    return {"workload": WORKLOAD, "pop": POP, "global_batch": BATCH, "max_nodes": N_MAX, "max_conns": C_MAX,
            "fill": FILL, "schema": "tanh/sum", "population_seed": POP_SEED, "n_gpus": world,
            "parallelism": f"dp{world} (genome blocks of one 10k population)",
            "l2": "flushed between timed steps (GPU arm)"}


def streaming_rooflines(net_bytes_c2=None, net_bytes_c5=None):
    """HBM rooflines of the streaming step kernels from the committed ncu
    summary (profiles/*_ncu_summary.json; cold-cache, serialised durations):
    DRAM bytes, the algorithmic bytes (genomes read + written), achieved
    GB/s and the fraction of the measured HBM peak.  C5 = pop 100k N128/C1024
    (37,888 B per genome), C2 = pop 10k N64/C256 (10,752 B)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu_summary.json")))
    if not files:
        return None
    d = json.load(open(files[-1]))
    peak, peak_src = hbm_peak()
    g5, g2 = 37_888, 10_752
    # kernel: (genome reads, genome writes, genome bytes, population, extra bytes written per genome)
    alg = {"step_c5_k_transform": (1, 0, g5, 100_000), "step_c5_k_crossover": (2, 1, g5, 100_000),
           "step_c5_k_mutate_apply": (1, 0, g5, 100_000), "step_c5_k_mutate_attrs": (1, 1, g5, 100_000),
           "k3_distance_c5": (1, 0, g5, 100_000), "k1_transform_c2": (1, 0, g2, 10_000),
           "step_c2_k_crossover": (2, 1, g2, 10_000), "step_c2_k_mutate_apply": (1, 0, g2, 10_000),
           "step_c2_k_mutate_attrs": (1, 1, g2, 10_000)}
    out = {}
    extra = {"step_c5_k_transform": net_bytes_c5 or 0, "k1_transform_c2": net_bytes_c2 or 0}  # K1 writes a NetLayout block
    for k, (r, w, gb, pop) in alg.items():
        v = d.get(k)
        if not v or "duration_us" not in v:
            continue
        t = v["duration_us"] * 1e-6
        a = (r + w) * gb * pop + extra.get(k, 0) * pop
        dram = v.get("dram_read", 0.0) + v.get("dram_write", 0.0)
        out[k] = {"ms": t * 1e3, "algorithmic_bytes": a, "dram_bytes": dram, "achieved_GBps": a / t / 1e9,
                  "frac_of_hbm": a / t / 1e9 / peak, "dram_over_algorithmic": dram / a if a else None}
    return {"source": os.path.relpath(files[-1], ROOT), "peak_GBps": peak, "peak_source": peak_src,
            "note": "algorithmic bytes = genomes read + written in the canonical FP64 layout (+ the NetLayout block "
                    "K1 writes); crossover reads two parents (elites read one), mutate_apply reads and rewrites only "
                    "structural edits; at C2 the population fits L2, so DRAM bytes can be below the algorithmic bytes",
            "kernels": out}


def cpu_info() -> dict:
    model, threads = None, os.cpu_count() or 1
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    if model is None:
        try:
            for line in open("/proc/cpuinfo"):
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
        except Exception:
            model = "unknown"
    return {"cpu_model": model, "host_threads": threads}


def loaded_native_libs() -> list:
    """Shared objects of this repo mapped into the process (evidence of which code ran)."""
    libs = set()
    try:
        for line in open("/proc/self/maps"):
            p = line.split()[-1]
            if p.endswith(".so") and (p.startswith(ROOT) or "/repo/" in p):
                libs.add(os.path.relpath(p, ROOT) if p.startswith(ROOT) else p)
    except Exception:
        pass
    return sorted(libs)


def ncu_traffic(name: str):
    """DRAM bytes per launch of a kernel from the newest committed ncu summary
    (profiles/*_ncu_summary.json, scripts/ncu_summary.py), or (None, None)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu_summary.json")))
    for f in reversed(files):
        try:
            d = json.load(open(f)).get(name)
        except Exception:
            continue
        if d and "dram_read" in d:
            return d["dram_read"] + d.get("dram_write", 0.0), os.path.relpath(f, ROOT)
    return None, None


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def hbm_peak():
    """(GB/s, source): the driver's measured copy bandwidth, else the recipe's
    fallback (B200_PROFILING.md: 6.65 TB/s, an earlier measurement on this pool)."""
    p = peaks().get("hbm_gbs")
    if p:
        return float(p), "of measured: MEASURED_PEAKS.json hbm_gbs (burst copy)"
    return 6650.0, "of fallback: B200_PROFILING.md 6.65 TB/s (MEASURED_PEAKS.json absent)"


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    r = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                        "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                    if r.returncode == 0 and r.stdout.strip():
                        self.samples.append([x.strip() for x in r.stdout.strip().split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 3 + i and s[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def _ref_tools():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as ol  # loads oracle/ libraries only
    return ol


def reference_population():
    syn = synthetic()
    nodes, conns = syn.synthetic_population(POP, N_MAX, C_MAX, FILL, NI, NO, seed=POP_SEED)
    X, Y = syn.regression_dataset(BATCH, NI, NO, seed=0)
    return nodes, conns, X, Y


def cpu_reference_step(ol, nodes, conns, X, Y, threads):
    """One step of the headline workload on the host: the reference's
    transform + batch_forward (network.hpp:122, 294; parallel_for over all
    threads) of the whole population, then the MSE fitness.  Returns seconds."""
    prob = ol.Problem(N_MAX, C_MAX, list(range(NI)), list(range(NI, NI + NO)))
    t0 = time.perf_counter()
    st, bad, msg, out = ol.ref_batch_forward(prob, ol.SchemaSpec(), nodes, conns, X, nthreads=threads)
    assert st == 0, msg
    _ = -np.mean((Y[None] - out) ** 2, axis=(1, 2))
    return time.perf_counter() - t0


def cpu_generation_reference(ol, nodes, conns, threads, forward_s):
    """SURVEY.md 8d / BASELINE.md 3: the reference's own operators for one
    generation of the C2 workload on the host: transform + batch_forward
    (timed by the caller, all threads), distance of every genome to S = 10
    representatives (parallel_for, all threads), crossover per slot and
    mutate per slot with one serial InnovationTable (one thread, as the
    reference's mutate contract requires).  Speciation / spawn / selection
    bookkeeping (O(P*S) integer work, no reference code) is not timed."""
    C = ol.C
    prob = ol.Problem(N_MAX, C_MAX, list(range(NI)), list(range(NI, NI + NO)))
    sh = prob.c()
    ref = ol.ref()
    P, S = nodes.shape[0], 10
    F64P = C.POINTER(C.c_double)
    reps_n, reps_c = np.ascontiguousarray(nodes[::P // S][:S]), np.ascontiguousarray(conns[::P // S][:S])
    out = np.empty((P, S))
    dc = ol.DistCfg(1.0, 0.5)
    t0 = time.perf_counter()
    ref.fr_distance_matrix(C.byref(sh), P, nodes.ctypes.data_as(F64P), conns.ctypes.data_as(F64P), S,
                           reps_n.ctypes.data_as(F64P), reps_c.ctypes.data_as(F64P), C.byref(dc), threads,
                           out.ctypes.data_as(F64P))
    t_dist = time.perf_counter() - t0
    keys = np.stack([ol.key_words(ol.key_split(ol.key_seed(5), i)) for i in range(P)]).astype(np.uint32)
    other = np.roll(np.arange(P), 1)
    on, oc = np.ascontiguousarray(nodes[other]), np.ascontiguousarray(conns[other])
    cn, cc = np.empty_like(nodes), np.empty_like(conns)
    t0 = time.perf_counter()
    ref.fr_crossover_population(C.byref(sh), P, nodes.ctypes.data_as(F64P), conns.ctypes.data_as(F64P),
                                on.ctypes.data_as(F64P), oc.ctypes.data_as(F64P),
                                keys.ctypes.data_as(C.POINTER(C.c_uint32)), cn.ctypes.data_as(F64P),
                                cc.ctypes.data_as(F64P))
    t_x = time.perf_counter() - t0
    t0 = time.perf_counter()
    st, bad, nk, mn, mc = ol.mutate_population(prob, ol.SchemaSpec(), cn, cc, keys, ol.mut_cfg(), 10_000,
                                               use_ref=True)
    t_m = time.perf_counter() - t0
    assert st == 0
    total = forward_s + t_dist + t_x + t_m
    return {"value": 1.0 / total, "unit": "generations/s", "ms_per_generation": total * 1e3, "kind": "reference",
            "cores": threads, **cpu_info(),
            "components_ms": {"transform_plus_batch_forward": forward_s * 1e3, "distance_x10_parallel_for": t_dist * 1e3,
                              "crossover_per_slot_1_thread": t_x * 1e3, "mutate_per_slot_serial_table": t_m * 1e3},
            "sample": f"full pop {P}: {P} x {S} distances, {P} crossovers, {P} mutations (paper defaults)"}


def c5_distance(dev, stream, flush, reps: int = 5, population: str = "random"):
    """K3 at C5 shapes: pop 100k, N128/C1024, S = 10
    representatives; HBM-bound, so reported against the measured HBM peak.
    population "random": 2,000 distinct synthetic genomes (random topologies:
    ~17% of a row's markers in any one representative) tiled to 100k on the
    device, representatives drawn from them; "lineage": 2,000 mutated copies
    of 10 ancestors (the representatives), the overlap a NEAT run's species
    have.  K3's cost depends on row counts and marker overlap, not values."""
    import torch
    import paper_2504_08339_b200 as fnb
    from paper_2504_08339_b200.synthetic import lineage_population, synthetic_population
    P5, N5, C5, S5, uniq = 100_000, 128, 1024, 10, 2_000
    if population == "lineage":
        n_h, c_h, rn_h, rc_h = lineage_population(uniq, N5, C5, ancestors=S5, fill=FILL, num_inputs=NI,
                                                  num_outputs=NO, seed=5)
    else:
        n_h, c_h = synthetic_population(uniq, N5, C5, FILL, NI, NO, seed=5)
        rn_h, rc_h = n_h[1::200][:S5], c_h[1::200][:S5]
    eng5 = fnb.Engine(fnb.GenomeLimits(N5, C5), list(range(NI)), list(range(NI, NI + NO)), fnb.AttributeSchema(),
                      device=dev.index)
    base_n, base_c = torch.from_numpy(n_h).to(dev), torch.from_numpy(c_h).to(dev)
    nodes5 = base_n.repeat(P5 // uniq, 1, 1).contiguous()
    conns5 = base_c.repeat(P5 // uniq, 1, 1).contiguous()
    del base_n, base_c
    rn = torch.from_numpy(np.ascontiguousarray(rn_h)).to(dev)
    rc = torch.from_numpy(np.ascontiguousarray(rc_h)).to(dev)
    out = torch.empty((P5, S5), dtype=torch.float64, device=dev)
    for _ in range(2):
        eng5.distance_d(nodes5, conns5, rn, rc, out, stream=stream)
    ms = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        eng5.distance_d(nodes5, conns5, rn, rc, out, stream=stream)
        b.record(stream)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    t = float(np.median(ms)) / 1e3
    alg = P5 * (40 * N5 + 32 * C5) + P5 * S5 * 8  # canonical genome bytes + distances out
    peak, peak_src = hbm_peak()
    achieved = alg / t / 1e9
    c5_traffic, c5_src = ncu_traffic("k3_distance_c5")
    del nodes5, conns5
    return {"workload": f"C5 K3 distance: pop 100k, N128/C1024, S=10 reps, fill 0.75, {population} population "
                        "(2k distinct genomes tiled)",
            "ms": t * 1e3, "genomes_per_s": P5 / t,
            "roofline": {"kernel": "K3 union-table build (6 kernels) + k_distance", "bound": "hbm", "achieved": achieved,
                         "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "algorithmic_bytes_per_launch": alg, "traffic": c5_traffic,
                         "traffic_source": c5_src,
                         "peak_source": peak_src}}


def c3_cppn(eng, nets, dev, stream, flush, reps: int = 3):
    """C3: the pop-10k C2 networks as CPPNs queried over a
    256 x 256 grid (x, y, r, bias) = 65,536 queries per genome, image-MSE
    fitness fused into the forward (outputs never materialised)."""
    import torch
    import paper_2504_08339_b200 as fnb
    from paper_2504_08339_b200.synthetic import cppn_dataset
    Xh, Yh = cppn_dataset(256)
    X = torch.from_numpy(Xh.astype(np.float32)).to(dev)
    Y = torch.from_numpy(Yh.astype(np.float32)).to(dev)
    fit = torch.empty(P_SHARD, dtype=torch.float64, device=dev)
    eng.forward_d(nets, P_SHARD, X, Y, fnb.FIT_NEG_MSE, 0.0, fitness=fit, stream=stream)
    ms = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        eng.forward_d(nets, P_SHARD, X, Y, fnb.FIT_NEG_MSE, 0.0, fitness=fit, stream=stream)
        b.record(stream)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    t = float(np.median(ms)) / 1e3
    return {"workload": "C3 CPPN: pop 10k (C2 networks), 256x256 grid = 65,536 queries per genome, image MSE",
            "forward_ms": t * 1e3, "evals_per_s": P_SHARD * Xh.shape[0] / t}


def c4_hyperneat(dev, stream, flush, reps: int = 3):
    """C4: pop 4k CPPNs (N32/C128) queried at the 28 x 8
    substrate connections, each policy run for 1000 steps of the synthetic
    27-obs / 8-act linear dynamics.  One step = K1 + K2 (224 queries per
    CPPN) + the rollout kernel."""
    import torch
    import paper_2504_08339_b200 as fnb
    from paper_2504_08339_b200.synthetic import CPPN_ACTS, cppn_population, hyper_dynamics
    P4 = 4000
    nodes_h, conns_h = cppn_population(P4, 32, 128, seed=4)
    A, B, s0 = hyper_dynamics(seed=4)
    eng4 = fnb.Engine(fnb.GenomeLimits(32, 128), [0, 1, 2, 3, 4], [5], fnb.AttributeSchema(CPPN_ACTS, ["sum"]),
                      device=dev.index)
    cfg = fnb.HyperConfig()
    nodes, conns = torch.from_numpy(nodes_h).to(dev), torch.from_numpy(conns_h).to(dev)
    f32 = lambda x: torch.from_numpy(x.astype(np.float32)).to(dev)
    dA, dB, ds0 = f32(A), f32(B), f32(s0)
    nets = eng4.alloc_nets(P4)
    fit = torch.empty(P4, dtype=torch.float64, device=dev)

    def run():
        eng4.transform_d(nodes, conns, nets, stream)
        eng4.hyper_evaluate_d(nets, P4, cfg, dA, dB, ds0, fit, stream=stream)

    run()
    ms = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        run()
        b.record(stream)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    t = float(np.median(ms)) / 1e3
    Q = (cfg.num_obs + 1) * cfg.num_act
    return {"workload": "C4 HyperNEAT: pop 4k CPPNs (N32/C128), 28x8 substrate queries, 27-obs/8-act policy, "
                        "1000-step linear-dynamics rollout",
            "ms": t * 1e3, "policy_steps_per_s": P4 * cfg.steps / t, "cppn_evals_per_s": P4 * Q / t,
            "generations_equiv_per_s": 1.0 / t}


def timed_generations(ev, X, Y, dev, flush, world: int, gens: int, warm: int, shard=None):
    """Mean device time of one generation (evaluate -> speciate -> stagnate ->
    spawn -> reproduce), CUDA events on the evolver stream, max over ranks.
    One GPU: fnb_evolve (one CUDA graph per generation, host reads RunStats
    each generation -- the loop a user runs).  N GPUs: the sharded step
    (distributed.ShardedEvolution).  The working set (two population buffers
    + nets) exceeds L2, and L2 is flushed before the timed run."""
    import torch
    import torch.distributed as dist
    es = torch.cuda.ExternalStream(ev.stream_handle(), device=dev)
    if shard is None:
        ev.run(X.cpu().double().numpy(), Y.cpu().double().numpy(), generation_limit=warm)
    else:
        for _ in range(warm):
            shard.generation()
    flush.zero_()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = ev.engine.launch_count
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(es)
    t0 = time.perf_counter()
    stats = None
    if shard is None:
        _, _, stats = ev.run(X.cpu().double().numpy(), Y.cpu().double().numpy(), generation_limit=gens)
    else:
        for _ in range(gens):
            shard.generation()
    b.record(es)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ms = a.elapsed_time(b) / gens
    if world > 1:
        t = torch.tensor([ms, wall], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, wall = (float(x) for x in t.tolist())
    out = {"ms_per_generation": ms, "generations_per_s": 1e3 / ms, "wall_s": wall, "generations_timed": gens,
           "launches_per_generation": (ev.engine.launch_count - launches0) / gens, "species": ev.state_species()}
    if shard is None:
        out["graph_mode"] = {2: "one CUDA graph per generation (conditional step node)",
                             1: "evaluate graph + step graph", 0: "eager"}.get(ev.run_mode(), "unknown")
        out["mean_host_ms_per_generation"] = float(np.mean([s.elapsed_ms for s in stats]))
    else:
        out.update(collectives_per_generation=shard.collectives / (warm + gens),
                   parents_exchanged_last=shard.parents_exchanged, sharding="population blocks (ShardedEvolution)")
    return out


def c5_generation(dev, flush, world: int = 1, rank: int = 0, gens: int = 4, warm: int = 2):
    """BASELINE config 5: the full device generation loop (K1+K2 evaluation,
    then speciate / stagnation / spawn / reproduce with K3, K5, K6, K7) at
    pop 100k, N128/C1024.  At N GPUs the population is sharded
    (ShardedEvolution: each rank evaluates, speciates and reproduces its own
    genome block).  The population starts as 2,000 distinct synthetic
    genomes tiled to 100k on the device."""
    import torch
    import paper_2504_08339_b200 as fnb
    from paper_2504_08339_b200.distributed import ShardedEvolution
    from paper_2504_08339_b200.evolve import Evolver, NeatConfig
    syn = synthetic()
    P5, N5, C5, uniq = 100_000, 128, 1024, 2_000
    n_h, c_h = syn.synthetic_population(uniq, N5, C5, FILL, NI, NO, seed=5)
    eng5 = fnb.Engine(fnb.GenomeLimits(N5, C5), list(range(NI)), list(range(NI, NI + NO)), fnb.AttributeSchema(),
                      device=dev.index)
    ev = Evolver(eng5, NeatConfig(pop_size=P5), seed=5)
    nodes = torch.from_numpy(n_h).to(dev).repeat(P5 // uniq, 1, 1)
    conns = torch.from_numpy(c_h).to(dev).repeat(P5 // uniq, 1, 1)
    ev.set_population_d(nodes, conns)
    del nodes, conns
    X_h, Y_h = syn.regression_dataset(BATCH, NI, NO, seed=0)
    X = torch.from_numpy(X_h.astype(np.float32)).to(dev)
    Y = torch.from_numpy(Y_h.astype(np.float32)).to(dev)
    shard = ShardedEvolution(ev, X, Y) if world > 1 else None
    r = timed_generations(ev, X, Y, dev, flush, world, gens, warm, shard)
    ev.close()
    return {"workload": f"C5 generation loop: pop 100k, N128/C1024, B=1024 func-fit, {world} GPU(s) "
                        "(2k distinct genomes tiled)", **r, "scaling": "strong", "timing": "max over ranks"}


def rich_schema(dev, stream, flush, reps: int = 5):
    """The generic forward (k_forward<SPT, -1, -1>: per-node activation and
    aggregation) on the C2 workload with the rich schema {identity, tanh,
    sigmoid, relu, sin} x {sum, product, max, mean}, seeds 0..2 of the
    population generator."""
    import torch
    import paper_2504_08339_b200 as fnb
    syn = synthetic()
    schema = fnb.AttributeSchema(["identity", "tanh", "sigmoid", "relu", "sin"], ["sum", "product", "max", "mean"])
    eng = fnb.Engine(fnb.GenomeLimits(N_MAX, C_MAX), list(range(NI)), list(range(NI, NI + NO)), schema,
                     device=dev.index)
    X_h, Y_h = syn.regression_dataset(BATCH, NI, NO, seed=0)
    X = torch.from_numpy(X_h.astype(np.float32)).to(dev)
    Y = torch.from_numpy(Y_h.astype(np.float32)).to(dev)
    out = {}
    for seed in range(3):
        n_h, c_h = syn.synthetic_population(POP, N_MAX, C_MAX, FILL, NI, NO, n_act=5, n_agg=4, seed=seed)
        nodes, conns = torch.from_numpy(n_h).to(dev), torch.from_numpy(c_h).to(dev)
        nets = eng.alloc_nets(POP)
        fit = torch.empty(POP, dtype=torch.float64, device=dev)

        def run():
            eng.transform_d(nodes, conns, nets, stream)
            eng.forward_d(nets, POP, X, Y, fnb.FIT_NEG_MSE, 0.0, fitness=fit, stream=stream)

        run()
        ms = []
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            run()
            b.record(stream)
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        t = float(np.median(ms)) / 1e3
        out[f"seed{seed}"] = {"transform_plus_forward_ms": t * 1e3, "evals_per_s": POP * BATCH / t}
    return {"workload": "C2 shapes, rich schema (5 activations x 4 aggregations per node), pop 10k, B=1024",
            **out}


def evolved_population(eng, dev, stream, flush, X, Y, gens: int = 100):
    """K1+K2 on an EVOLVED pop-10k population (100 generations
    of the device loop from minimal genomes on the C2 func-fit data) -- the
    topologies a NEAT run actually evaluates, next to the synthetic fill-0.75
    headline."""
    import torch
    import paper_2504_08339_b200 as fnb
    from paper_2504_08339_b200.evolve import Evolver, NeatConfig
    ev = Evolver(eng, NeatConfig(pop_size=P_SHARD), seed=7)
    ev.init_population()
    es = torch.cuda.ExternalStream(ev.stream_handle())
    t0 = time.perf_counter()
    for _ in range(gens):
        ev.evaluate_d(X, Y)
        ev.step()
    es.synchronize()
    loop_s = time.perf_counter() - t0
    n_ptr, c_ptr, _, _ = ev.device_state()
    nh, ch = ev.population()
    ev.close()
    nodes, conns = torch.from_numpy(nh).to(dev), torch.from_numpy(ch).to(dev)
    nets = eng.alloc_nets(P_SHARD)
    fit = torch.empty(P_SHARD, dtype=torch.float64, device=dev)

    def run():
        eng.transform_d(nodes, conns, nets, stream)
        eng.forward_d(nets, P_SHARD, X, Y, fnb.FIT_NEG_MSE, 0.0, fitness=fit, stream=stream)

    run()
    ms = []
    for _ in range(5):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        run()
        b.record(stream)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    t = float(np.median(ms)) / 1e3
    n_nodes = float(np.mean(np.sum(~np.isnan(nh[:, :, 0]), axis=1)))
    n_en = float(np.mean(np.sum(ch[:, :, 2] == 1.0, axis=1)))
    return {"workload": f"pop 10k after {gens} device generations from minimal genomes (C2 data, N64/C256)",
            "mean_nodes": n_nodes, "mean_enabled_conns": n_en, "transform_plus_forward_ms": t * 1e3,
            "evals_per_s": P_SHARD * BATCH / t, "wall_s_100_generations": loop_s}


def reference_arm(args, rank: int):
    """--impl reference: the reference's own CPU path on the box's host cores,
    the full workload every step (no extrapolation), W real warm-up steps."""
    if rank != 0:
        return
    ol = _ref_tools()
    if not ol.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref (the compiled reference) is missing"}))
        return
    threads = os.cpu_count() or 1
    nodes, conns, X, Y = reference_population()
    for _ in range(args.warmup):
        cpu_reference_step(ol, nodes, conns, X, Y, threads)
    ts = [cpu_reference_step(ol, nodes, conns, X, Y, threads) for _ in range(max(1, args.steps))]
    ms = float(np.mean(ts)) * 1e3
    v = POP * BATCH / (ms / 1e3)
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(args.gpus),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference", **cpu_info(),
                             "sample": f"full workload every step: {POP} genomes x {BATCH} samples, "
                                       "transform + batch_forward (parallel_for, grain 16) + MSE"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "native_so_loaded": loaded_native_libs()}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-generations", action="store_true")
    ap.add_argument("--no-c5", action="store_true", help="skip the C3 (CPPN), C4 (HyperNEAT) and C5 (pop 100k) measurements")
    ap.add_argument("--spt", type=int, default=0, help="forward columns per thread (tuning; 0 = auto)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        reference_arm(args, rank)
        return

    import torch
    import torch.distributed as dist
    import paper_2504_08339_b200 as fnb
    from paper_2504_08339_b200.distributed import shard_bounds

    if args.spt:
        fnb._native.lib().fnb_set_forward_spt(args.spt)
    # FNB_BENCH_ONE_GPU=1 (test hook): every rank on cuda:0 over gloo, to run the
    # N>1 orchestration on a one-GPU box; numbers from it are not bench values
    one_gpu = os.environ.get("FNB_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    syn = synthetic()
    # the job's population: one pop-10k population, rank r holds genome block [lo, hi)
    all_n, all_c = syn.synthetic_population(POP, N_MAX, C_MAX, FILL, NI, NO, seed=POP_SEED)
    lo, hi = shard_bounds(POP, world, rank)
    nodes_h, conns_h = np.ascontiguousarray(all_n[lo:hi]), np.ascontiguousarray(all_c[lo:hi])
    PL = hi - lo
    X_h, Y_h = syn.regression_dataset(BATCH, NI, NO, seed=0)
    eng = fnb.Engine(fnb.GenomeLimits(N_MAX, C_MAX), list(range(NI)), list(range(NI, NI + NO)),
                     fnb.AttributeSchema(), device=local)
    X = torch.from_numpy(X_h.astype(np.float32)).to(dev)
    Y = torch.from_numpy(Y_h.astype(np.float32)).to(dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream()
    shard_max = max(shard_bounds(POP, world, r)[1] - shard_bounds(POP, world, r)[0] for r in range(world))

    def timed_eval(nodes_h, conns_h, steps, warmup):
        """K1 + K2 of this rank's genomes + the fitness all-gather, CUDA events, max over ranks."""
        P = nodes_h.shape[0]
        nodes = torch.from_numpy(nodes_h).to(dev)
        conns = torch.from_numpy(conns_h).to(dev)
        nets = eng.alloc_nets(P)
        pad = max(P, shard_max) if world > 1 else P
        fit = torch.zeros(pad, dtype=torch.float64, device=dev)
        fit_all = torch.empty(pad * world, dtype=torch.float64, device=dev)

        def step(ev=None):
            eng.transform_d(nodes, conns, nets, stream)
            if ev is not None:
                ev[0].record(stream)
            eng.forward_d(nets, P, X, Y, fnb.FIT_NEG_MSE, 0.0, fitness=fit, stream=stream)
            if ev is not None:
                ev[1].record(stream)
            if world > 1:
                dist.all_gather_into_tensor(fit_all, fit)

        step()
        eng.check_nets_d(nodes, conns, nets)  # correctness gate once, outside timing
        for _ in range(max(3, warmup)):
            flush.zero_()
            step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        launches0 = eng.launch_count
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        torch.cuda.synchronize()
        for i in range(steps):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            starts[i].record(stream)
            step(kev[i])
            ends[i].record(stream)
        torch.cuda.synchronize()
        launches = eng.launch_count - launches0
        tot = float(sum(s.elapsed_time(e) for s, e in zip(starts, ends)))
        fwd = float(np.mean([a.elapsed_time(b) for a, b in kev]))
        if world > 1:
            t = torch.tensor([tot], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tot = float(t.item())
            dist.barrier()
        del nodes, conns, nets
        return tot / steps, fwd, launches

    sampler = ClockSampler(local)
    sampler.start()
    ms_per_step, fwd_ms, launches = timed_eval(nodes_h, conns_h, args.steps, args.warmup)
    clocks = sampler.stop()
    value = POP * BATCH / (ms_per_step / 1e3)
    weak = None
    if world > 1:  # every rank a full 10k population of its own
        wn, wc = syn.synthetic_population(P_SHARD, N_MAX, C_MAX, FILL, NI, NO, seed=POP_SEED + rank)
        w_ms, _, _ = timed_eval(wn, wc, args.steps, args.warmup)
        weak = {"value": P_SHARD * world * BATCH / (w_ms / 1e3), "unit": UNIT, "ms_per_step": w_ms,
                "scaling": "weak", "pop_per_gpu": P_SHARD}
        del wn, wc

    # ---- e2e through the public host API (H2D + D2H inside every call) ----
    def e2e(pinned: bool):
        if pinned:
            pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
            n_, c_, x_, y_ = pin(nodes_h), pin(conns_h), pin(X_h), pin(Y_h)
        else:
            n_, c_, x_, y_ = nodes_h, conns_h, X_h, Y_h
        eng.evaluate(n_, c_, x_, y_, fnb.FIT_NEG_MSE)
        ts = []
        for _ in range(max(5, min(args.steps, 20))):
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            f_ = eng.evaluate(n_, c_, x_, y_, fnb.FIT_NEG_MSE)
            ts.append(time.perf_counter() - t0)
        t = float(np.median(ts))
        if world > 1:
            tt = torch.tensor([t], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = float(tt.item())
        return t, f_.nbytes

    e2e_s, d2h = e2e(True)
    e2e_pageable_s, _ = e2e(False)
    h2d = nodes_h.nbytes + conns_h.nbytes + X_h.nbytes + Y_h.nbytes

    # ---- generations/s of the pop-10k loop ----
    def section(fn, *a):
        """A secondary measurement; its failure is reported, never fatal to the headline line."""
        try:
            return fn(*a)
        except Exception as e:  # noqa: BLE001
            return {"error": repr(e)[:300]}

    def generations_c2():
        from paper_2504_08339_b200.distributed import ShardedEvolution
        from paper_2504_08339_b200.evolve import Evolver, NeatConfig
        ev = Evolver(eng, NeatConfig(pop_size=POP), seed=POP_SEED)
        ev.set_population(all_n, all_c)
        shard = ShardedEvolution(ev, X, Y) if world > 1 else None
        g = timed_generations(ev, X, Y, dev, flush, world, max(5, args.steps), max(3, args.warmup), shard)
        g.update(scaling="strong", note="one pop-10k population per job, C2 shapes, B=1024 func-fit; max over ranks")
        ev.close()
        return g

    gen = None if args.no_generations else section(generations_c2)

    c3 = c4 = c5 = c5l = c5g = evo = rich = None
    if rank == 0 and world == 1 and not args.no_c5:
        nets10 = eng.alloc_nets(POP)
        eng.transform_d(torch.from_numpy(all_n).to(dev), torch.from_numpy(all_c).to(dev), nets10, stream)
        c3 = section(c3_cppn, eng, nets10, dev, stream, flush)
        del nets10
        c4 = section(c4_hyperneat, dev, stream, flush)
        c5 = section(c5_distance, dev, stream, flush)
        c5l = section(c5_distance, dev, stream, flush, 5, "lineage")
        rich = section(rich_schema, dev, stream, flush)
    if not args.no_c5:
        c5g = section(c5_generation, dev, flush, world, rank)
    if rank == 0 and world == 1 and not args.no_generations:
        evo = section(evolved_population, eng, dev, stream, flush, X, Y)

    # ---- roofline for the dominant kernel (K2 forward, this rank's genomes) ----
    k2_traffic, k2_traffic_src = ncu_traffic("k2_forward_main_pass")
    n_en = int(np.sum(conns_h[:, :, 2] == 1.0))
    n_ops = int(np.sum(~np.isnan(nodes_h[:, :, 0]))) - PL * NI
    flops = 2.0 * BATCH * (n_en + n_ops)          # FMA per enabled edge + resp*agg+bias per node
    fwd_s = fwd_ms / 1e3
    pk = peaks()
    sm_clock = (pk.get("sm_max_mhz") or 1965.0) * 1e6
    fp32_peak = 148 * 128 * 2 * sm_clock / 1e12
    smem_bytes = 4.0 * BATCH * (n_en + n_ops)     # one 4-byte LDS per edge-sample, one STS per node-sample
    smem_peak = 148 * 128 * sm_clock / 1e12       # TB/s (128 B/clk/SM)
    smem_ach = smem_bytes / fwd_s / 1e12

    cpu = cpu_gen = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            ol = _ref_tools()
            if ol.ref_available():
                threads = os.cpu_count() or 1
                rn, rc, rX, rY = reference_population()
                cpu_reference_step(ol, rn, rc, rX, rY, threads)  # warm
                t_fwd = cpu_reference_step(ol, rn, rc, rX, rY, threads)
                cpu = {"value": POP * BATCH / t_fwd, "unit": UNIT, "cores": threads, "kind": "reference",
                       **cpu_info(), "sample": f"full workload: {POP} genomes x {BATCH} samples, transform + "
                                               "batch_forward (parallel_for, grain 16) + MSE, one timed step"}
                cpu_gen = cpu_generation_reference(ol, rn, rc, threads, t_fwd)
            else:
                cpu = {"value": None, "error": "oracle/_ref missing"}
        except Exception as e:  # reported, never silently substituted
            cpu = {"value": None, "error": repr(e)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32 (forward), f64 (fitness)", "data": "synthetic",
            "config": config_dict(world),
            "e2e": {"value": POP * BATCH / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "api": "fnb_evaluate (host buffers, pinned)",
                    "h2d_gbps_effective": h2d / e2e_s / 1e9, "timing": "median of calls, max over ranks",
                    "pageable": {"value": POP * BATCH / e2e_pageable_s, "unit": UNIT,
                                 "api": "fnb_evaluate from pageable host memory (std::vector-like)"}},
            "gpu_launches": int(launches),
            "kernels": {"transform_plus_forward_ms": ms_per_step, "forward_ms": fwd_ms,
                        "transform_ms": ms_per_step - fwd_ms, "genomes_on_rank0": PL},
            "roofline": {"kernel": "k_forward (K2)", "bound": "smem", "achieved": smem_ach, "peak": smem_peak,
                         "unit": "TB/s", "frac": smem_ach / smem_peak, "traffic": k2_traffic,
                         "traffic_source": k2_traffic_src,
                         "algorithmic": "4 B LDS per enabled edge x sample + 4 B per node x sample",
                         "peak_source": "128 B/clk/SM x 148 SMs at MEASURED_PEAKS sm_max_mhz",
                         "fp32": {"achieved_TFLOPs": flops / fwd_s / 1e12, "peak_TFLOPs": fp32_peak,
                                  "frac": flops / fwd_s / 1e12 / fp32_peak}},
            "clocks": clocks,
        }
        for k, v in (("weak_scaling", weak), ("generations", gen), ("c5_distance", c5), ("c5_distance_lineage", c5l),
                     ("c3_cppn", c3), ("c4_hyperneat", c4), ("evolved", evo), ("c5_generation", c5g),
                     ("rich_schema", rich),
                     ("cpu_baseline", cpu)):
            if v is not None:
                line[k] = v
        if cpu_gen is not None and gen is not None and "error" not in gen:
            gen["cpu_baseline"] = cpu_gen
        nb5 = fnb.Engine(fnb.GenomeLimits(128, 1024), list(range(NI)), list(range(NI, NI + NO)), fnb.AttributeSchema(),
                         device=local).net_bytes
        sr = streaming_rooflines(eng.net_bytes, nb5)
        if sr is not None:
            line["streaming_rooflines"] = sr
        line["native_so_loaded"] = loaded_native_libs()
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
