"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

    python scripts/summarize_launches.py gpurun_out/launches10.csv > profiles/r01_launches.txt
"""
import collections
import csv
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in data:
        if not r[vi]:
            continue
        name = r[ki].split("(")[0].strip()[:70]
        us = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(a[1] for a in agg.values())
    print(f"# {path}: {len(data)} launches, {tot:.1f} us total (cold-cache, serialised by ncu)")
    print(f"{'total_us':>10} {'share':>6} {'n':>5} {'us/launch':>10}  kernel")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t:10.1f} {t / tot:6.1%} {n:5d} {t / n:10.1f}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
