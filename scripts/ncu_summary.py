"""Summarise `ncu --set full` reports into one JSON (committed under profiles/).

    python scripts/ncu_summary.py profiles/r01_ncu_summary.json name=gpurun_out/x.ncu-rep ...

Per kernel: duration, DRAM bytes read/written (the `traffic` of bench.py's
roofline objects), instructions, issue-slot utilisation, occupancy, IPC.
"""
import csv
import json
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_slots_busy_pct",
    "sm__inst_executed.avg.per_cycle_active": "ipc_active",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "registers",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1tex_throughput_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "nsecond": 1e-9}


def summarise_all(path):
    """One summary per kernel launch captured in the report."""
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return [summarise_row(rows[0], rows[1], vals) for vals in rows[2:]]


def summarise(path):
    return summarise_all(path)[0]


def summarise_row(hdr, units, vals):
    d = {"kernel": vals[hdr.index("Kernel Name")].split("(")[0]}
    for m, name in METRICS.items():
        if m in hdr:
            i = hdr.index(m)
            try:
                v = float(vals[i].replace(",", ""))
            except ValueError:
                continue
            d[name] = v * SCALE.get(units[i], 1.0)
    if "duration" in d:
        d["duration_us"] = d.pop("duration") * 1e6
    return d


def main():
    dst = sys.argv[1]
    res = {}
    for arg in sys.argv[2:]:
        name, path = arg.split("=", 1)
        if name.endswith("*"):  # every launch in the report: name + kernel
            for d in summarise_all(path):
                res[name[:-1] + d["kernel"].split("<")[0].split("::")[-1].replace("void ", "").strip()] = d
        else:
            res[name] = summarise(path)
    json.dump(res, open(dst, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
