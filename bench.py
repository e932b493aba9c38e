"""Benchmark: network evals/s of the NEAT evaluation step at BASELINE config 2.

One step = transform (K1) + forward with the fused func-fit fitness (K2) of a
10k-genome shard (N_max=64, C_max=256, fill 0.75, tanh/sum) over a
1024-sample batch, plus the fitness all-gather across ranks (the real
per-generation exchange).  Weak scaling: every rank owns a 10k shard, so the
job evaluates 10k*N genomes per step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Rank 0 prints one JSON line.  --impl reference times the reference's own CPU
path (oracle/_ref = the unmodified reference headers, all host threads) on a
bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
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
P_SHARD, N_MAX, C_MAX, FILL, BATCH, NI, NO = 10_000, 64, 256, 0.75, 1024, 4, 1
WORKLOAD = "C2 func-regression: pop 10k per GPU, B=1024, N_max=64, C_max=256, fill 0.75, tanh/sum"


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


def cpu_reference(P_sample: int, seed: int = 0, target_s: float = 8.0):
    """Reference batch_forward (transform + forward, network.hpp:122/294) on all host cores via oracle/_ref."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as ol
    from paper_2504_08339_b200.synthetic import regression_dataset, synthetic_population
    if ol.ref_available():
        kind = "reference"
    else:
        kind = "port"
    threads = os.cpu_count() or 1
    prob = ol.Problem(N_MAX, C_MAX, list(range(NI)), list(range(NI, NI + NO)))
    schema = ol.SchemaSpec()
    X, Y = regression_dataset(BATCH, NI, NO, seed=seed)

    def run(P):
        nodes, conns = synthetic_population(P, N_MAX, C_MAX, FILL, NI, NO, seed=seed)
        t0 = time.perf_counter()
        if kind == "reference":
            st, bad, msg, out = ol.ref_batch_forward(prob, schema, nodes, conns, X, nthreads=threads)
            assert st == 0, msg
        else:
            for p in range(P):
                net = ol.oracle_transform(prob, schema, nodes[p], conns[p])
                out = ol.oracle_forward(prob, schema, nodes[p], net, X)
        _ = -np.mean((Y[None] - out) ** 2, axis=(1, 2)) if out.ndim == 3 else None
        return time.perf_counter() - t0

    probe = max(threads * 4, 64)
    dt = run(probe)
    P = int(min(P_sample or 10**9, max(probe, probe * target_s / max(dt, 1e-6))))
    P = min(P, P_SHARD)
    dt = run(P)
    return {"value": P * BATCH / dt, "unit": UNIT, "cores": threads if kind == "reference" else 1, "kind": kind,
            "sample": f"{P} genomes x {BATCH} samples of the C2 workload, transform+forward+MSE, {dt:.2f} s"}


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


def c5_generation(dev, flush, world: int = 1, gens: int = 4, warm: int = 2):
    """BASELINE config 5: the full device generation loop (K1+K2 evaluation,
    then speciate / stagnation / spawn / reproduce with K3, K5, K6, K7) at
    pop 100k, N128/C1024, sharded over the job's GPUs: evaluation by genome
    blocks with the fitness all-gather, and at N > 1 the reproduction too
    (distributed.py shard_step: children [lo, hi) per rank, then an
    all-gather of the next population).  The population starts as 2,000
    distinct synthetic genomes tiled to 100k on the device."""
    import torch
    import torch.distributed as dist
    import paper_2504_08339_b200 as fnb
    from paper_2504_08339_b200.distributed import DeviceShardBackend, ShardedGeneration
    from paper_2504_08339_b200.evolve import Evolver, NeatConfig
    from paper_2504_08339_b200.synthetic import regression_dataset, synthetic_population
    P5, N5, C5, uniq = 100_000, 128, 1024, 2_000
    n_h, c_h = synthetic_population(uniq, N5, C5, FILL, NI, NO, seed=5)
    eng5 = fnb.Engine(fnb.GenomeLimits(N5, C5), list(range(NI)), list(range(NI, NI + NO)), fnb.AttributeSchema(),
                      device=dev.index)
    ev = Evolver(eng5, NeatConfig(pop_size=P5), seed=5)
    nodes = torch.from_numpy(n_h).to(dev).repeat(P5 // uniq, 1, 1)
    conns = torch.from_numpy(c_h).to(dev).repeat(P5 // uniq, 1, 1)
    ev.set_population_d(nodes, conns)
    del nodes, conns
    X_h, Y_h = regression_dataset(BATCH, NI, NO, seed=0)
    X = torch.from_numpy(X_h.astype(np.float32)).to(dev)
    Y = torch.from_numpy(Y_h.astype(np.float32)).to(dev)
    sg = ShardedGeneration(DeviceShardBackend(ev, X, Y), shard_step=True)
    es = sg.backend.stream
    gms, ems = [], []
    for it in range(warm + gens):
        flush.zero_()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(es)
        sg.evaluate()
        e1.record(es)
        if world > 1:
            sg.reproduce_sharded()
        else:
            ev.step()
        e2.record(es)
        torch.cuda.synchronize()
        if it >= warm:
            gms.append(e0.elapsed_time(e2))
            ems.append(e0.elapsed_time(e1))
    g_ms, e_ms = float(np.mean(gms)), float(np.mean(ems))
    if world > 1:
        t = torch.tensor([g_ms, e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        g_ms, e_ms = (float(x) for x in t.tolist())
    agree = sg.replicas_agree()
    sp = ev.species()
    ev.close()
    return {"workload": f"C5 generation loop: pop 100k, N128/C1024, B=1024 func-fit, {world} GPU(s) "
                        "(2k distinct genomes tiled)",
            "ms_per_generation": g_ms, "generations_per_s": 1e3 / g_ms, "evaluate_ms": e_ms, "evolve_step_ms": g_ms - e_ms,
            "evals_per_s": P5 * BATCH / (e_ms / 1e3), "species": int(sp["count"]), "generations_timed": gens,
            "sharding": "evaluation + reproduction by genome blocks" if world > 1 else "single GPU",
            "replicas_agree": bool(agree), "scaling": "strong", "timing": "max over ranks"}


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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-generations", action="store_true")
    ap.add_argument("--no-c5", action="store_true", help="skip the C3 (CPPN), C4 (HyperNEAT) and C5 (pop 100k K3 distance) measurements")
    ap.add_argument("--spt", type=int, default=0, help="forward columns per thread (tuning; 0 = auto)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return
        vals = []
        for _ in range(args.warmup):
            pass
        base = None
        for _ in range(max(1, args.steps)):
            base = cpu_reference(0, target_s=max(1.0, 20.0 / max(1, args.steps)))
            vals.append(base["value"])
        v = float(np.median(vals))
        line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": P_SHARD * BATCH / v * 1e3,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": {"workload": WORKLOAD, "global_batch": BATCH, "pop": P_SHARD},
                "cpu_baseline": {**base, "value": v},
                "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch
    import torch.distributed as dist
    import paper_2504_08339_b200 as fnb
    from paper_2504_08339_b200.synthetic import regression_dataset, synthetic_population

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

    nodes_h, conns_h = synthetic_population(P_SHARD, N_MAX, C_MAX, FILL, NI, NO, seed=1000 + rank)
    X_h, Y_h = regression_dataset(BATCH, NI, NO, seed=0)
    eng = fnb.Engine(fnb.GenomeLimits(N_MAX, C_MAX), list(range(NI)), list(range(NI, NI + NO)),
                     fnb.AttributeSchema(), device=local)
    nodes = torch.from_numpy(nodes_h).to(dev)
    conns = torch.from_numpy(conns_h).to(dev)
    X = torch.from_numpy(X_h.astype(np.float32)).to(dev)
    Y = torch.from_numpy(Y_h.astype(np.float32)).to(dev)
    nets = eng.alloc_nets(P_SHARD)
    fit = torch.empty(P_SHARD, dtype=torch.float64, device=dev)
    fit_all = torch.empty(P_SHARD * world, dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream()

    def step(ev=None):
        eng.transform_d(nodes, conns, nets, stream)
        if ev is not None:
            ev[0].record(stream)
        eng.forward_d(nets, P_SHARD, X, Y, fnb.FIT_NEG_MSE, 0.0, fitness=fit, stream=stream)
        if ev is not None:
            ev[1].record(stream)
        if world > 1:
            dist.all_gather_into_tensor(fit_all, fit)

    # correctness gate once, outside timing
    step()
    eng.check_nets_d(nodes, conns, nets)
    for _ in range(max(3, args.warmup)):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    sampler = ClockSampler(local)
    sampler.start()
    launches0 = eng.launch_count
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.zero_()  # L2 flush between timed steps (outside the events)
        starts[i].record(stream)
        step(kev[i])
        ends[i].record(stream)
    torch.cuda.synchronize()
    launches = eng.launch_count - launches0
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    fwd_ms = [a.elapsed_time(b) for a, b in kev]
    tot_ms = float(sum(step_ms))
    if world > 1:
        t = torch.tensor([tot_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
        dist.barrier()
    clocks = sampler.stop()
    ms_per_step = tot_ms / args.steps
    value = P_SHARD * world * BATCH / (ms_per_step / 1e3)

    # ---- e2e through the public host API (pinned host buffers, H2D + D2H inside) ----
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    nodes_p, conns_p, X_p, Y_p = pin(nodes_h), pin(conns_h), pin(X_h), pin(Y_h)
    eng.evaluate(nodes_p, conns_p, X_p, Y_p, fnb.FIT_NEG_MSE)
    e2e_steps = max(5, min(args.steps, 20))
    e2e_t = []
    for _ in range(e2e_steps):
        t0 = time.perf_counter()
        fit_h = eng.evaluate(nodes_p, conns_p, X_p, Y_p, fnb.FIT_NEG_MSE)
        e2e_t.append(time.perf_counter() - t0)
    e2e_s = float(np.median(e2e_t))  # per-call wall time (a call ends with its D2H + sync)
    if world > 1:
        t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    h2d = nodes_h.nbytes + conns_h.nbytes + X_h.nbytes + Y_h.nbytes
    d2h = fit_h.nbytes

    # ---- generations/s: evaluate + speciate/stagnate/spawn/reproduce on the device ----
    gen = None
    if not args.no_generations:
        # one 10k population for the whole job: replicated on every rank,
        # evaluation sharded, fitness all-gathered (distributed.py)
        from paper_2504_08339_b200.distributed import DeviceShardBackend, ShardedGeneration
        from paper_2504_08339_b200.evolve import Evolver, NeatConfig
        ev = Evolver(eng, NeatConfig(pop_size=P_SHARD), seed=1000)
        gn_h, gc_h = (nodes_h, conns_h) if rank == 0 else synthetic_population(P_SHARD, N_MAX, C_MAX, FILL, NI, NO,
                                                                                 seed=1000)
        ev.set_population(gn_h, gc_h)
        sg = ShardedGeneration(DeviceShardBackend(ev, X, Y))
        es = sg.backend.stream
        g_warm, g_steps = max(3, args.warmup), max(5, args.steps)
        gms, ems = [], []
        launches_g0 = 0
        for it in range(g_warm + g_steps):
            flush.zero_()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            if it == g_warm:
                launches_g0 = eng.launch_count
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(es)
            sg.evaluate()
            e1.record(es)
            ev.step()
            e2.record(es)
            es.synchronize()
            if it >= g_warm:
                gms.append(e0.elapsed_time(e2))
                ems.append(e0.elapsed_time(e1))
        g_ms, e_ms = float(np.mean(gms)), float(np.mean(ems))
        if world > 1:
            t = torch.tensor([g_ms, e_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            g_ms, e_ms = (float(x) for x in t.tolist())
        agree = sg.replicas_agree()
        sp = ev.species()
        gen = {"generations_per_s": 1e3 / g_ms, "ms_per_generation": g_ms,
               "evaluate_ms": e_ms, "evolve_step_ms": g_ms - e_ms,
               "generations_timed": g_steps, "species": int(sp["count"]),
               "launches_per_generation": (eng.launch_count - launches_g0) / g_steps,
               "replicas_agree": bool(agree), "scaling": "strong",
               "note": "one pop-10k population per job, C2 shapes; evaluation sharded over ranks + fitness "
                       "all-gather, step (speciate+stagnation+spawn+reproduce: K3,K5,K6,K7 + selection) replicated; "
                       "max over ranks"}
        ev.close()

    def section(fn, *a):
        """A secondary measurement; its failure is reported, never fatal to the headline line."""
        try:
            return fn(*a)
        except Exception as e:  # noqa: BLE001
            return {"error": repr(e)[:300]}

    c3 = section(c3_cppn, eng, nets, dev, stream, flush) if not args.no_c5 else None
    c4 = section(c4_hyperneat, dev, stream, flush) if not args.no_c5 else None
    evo = section(evolved_population, eng, dev, stream, flush, X, Y) if not args.no_generations else None
    c5g = section(c5_generation, dev, flush, world) if not args.no_c5 else None
    c5 = section(c5_distance, dev, stream, flush) if not args.no_c5 else None
    c5l = section(c5_distance, dev, stream, flush, 5, "lineage") if not args.no_c5 else None

    # ---- roofline for the dominant kernel (K2 forward) ----
    k2_traffic, k2_traffic_src = ncu_traffic("k2_forward_main_pass")
    n_en = int(np.sum(conns_h[:, :, 2] == 1.0))
    n_ops = int(np.sum(~np.isnan(nodes_h[:, :, 0]))) - P_SHARD * NI
    flops = 2.0 * BATCH * (n_en + n_ops)          # FMA per enabled edge + resp*agg+bias per node
    fwd_s = float(np.mean(fwd_ms)) / 1e3
    pk = peaks()
    sm_clock = (pk.get("sm_max_mhz") or 1965.0) * 1e6
    fp32_peak = 148 * 128 * 2 * sm_clock / 1e12
    achieved = flops / fwd_s / 1e12
    smem_bytes = 4.0 * BATCH * (n_en + n_ops)     # one 4-byte LDS per edge-sample, one STS per node-sample
    smem_peak = 148 * 128 * sm_clock / 1e12       # TB/s (128 B/clk/SM)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference(0)
        except Exception as e:  # reported, never silently substituted
            cpu = {"value": None, "error": repr(e)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32 (forward), f64 (fitness)", "data": "synthetic",
            "config": {"workload": WORKLOAD, "pop_per_gpu": P_SHARD, "global_pop": P_SHARD * world,
                       "global_batch": BATCH, "max_nodes": N_MAX, "max_conns": C_MAX, "fill": FILL,
                       "parallelism": f"dp{world} (population shards)", "l2": "flushed between timed steps"},
            "e2e": {"value": P_SHARD * world * BATCH / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "api": "fnb_evaluate (host buffers, pinned)",
                    "h2d_gbps_effective": h2d / e2e_s / 1e9, "timing": f"median of {e2e_steps} calls"},
            "gpu_launches": int(launches),
            "kernels": {"transform_plus_forward_ms": ms_per_step, "forward_ms": fwd_s * 1e3,
                        "transform_ms": ms_per_step - fwd_s * 1e3},
            "roofline": {"kernel": "k_forward (K2)", "bound": "fp32", "achieved": achieved, "peak": fp32_peak,
                         "unit": "TFLOP/s", "frac": achieved / fp32_peak, "traffic": k2_traffic,
                         "traffic_source": k2_traffic_src,
                         "peak_source": "nominal FP32 FMA peak at MEASURED_PEAKS sm_max_mhz (no measured FP32 peak)",
                         "smem": {"achieved_TBps": smem_bytes / fwd_s / 1e12, "peak_TBps": smem_peak,
                                  "frac": smem_bytes / fwd_s / 1e12 / smem_peak}},
            "clocks": clocks,
        }
        if gen is not None:
            line["generations"] = gen
        if c5 is not None:
            line["c5_distance"] = c5
        if c5l is not None:
            line["c5_distance_lineage"] = c5l
        if c3 is not None:
            line["c3_cppn"] = c3
        if c4 is not None:
            line["c4_hyperneat"] = c4
        if evo is not None:
            line["evolved"] = evo
        if c5g is not None:
            line["c5_generation"] = c5g
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
