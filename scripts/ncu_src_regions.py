"""Instruction / stall-sample shares of an ncu source CSV by file and by line range.

    python scripts/ncu_src_regions.py src.csv file.cu:a-b:name ...
"""
import collections
import csv
import os
import sys


def main(path, regions):
    rows = list(csv.reader(open(path)))
    cur = hdr = None
    agg, aggs = collections.Counter(), collections.Counter()
    lines, liness = collections.Counter(), collections.Counter()
    for r in rows:
        if r and r[0] == "File Path":
            cur = os.path.basename(r[1])
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8 or not r[0]:
            continue
        try:
            s = int(r[4]) if r[4] not in ("-", "") else 0
            i = int(r[7]) if r[7] not in ("-", "") else 0
        except ValueError:
            continue
        agg[cur] += i
        aggs[cur] += s
        lines[(cur, int(r[0]))] += i
        liness[(cur, int(r[0]))] += s
    T, TS = sum(agg.values()) or 1, sum(aggs.values()) or 1
    print(f"{path}: {T / 1e6:.0f} M warp instructions")
    for k in agg:
        print(f"  {k:28s} inst {100 * agg[k] / T:5.1f}%  samples {100 * aggs[k] / TS:5.1f}%")
    for spec in regions:
        f, rng, name = spec.split(":")
        a, b = map(int, rng.split("-"))
        i = sum(v for (ff, l), v in lines.items() if ff == f and a <= l <= b)
        s = sum(v for (ff, l), v in liness.items() if ff == f and a <= l <= b)
        print(f"  {name:28s} inst {100 * i / T:5.1f}%  samples {100 * s / TS:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
