"""Top CUDA source lines of an ncu report (--page source --print-source cuda,sass --csv).

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python scripts/ncu_source_hotspots.py src.csv [top]
"""
import csv
import os
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    cur, hdr, out = None, None, []
    for r in rows:
        if r and r[0] == "File Path":
            cur = os.path.basename(r[1])
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r or not r[0]:
            continue
        try:
            samples = int(r[4]) if r[4] not in ("-", "") else 0
            inst = int(r[7]) if r[7] not in ("-", "") else 0
        except (ValueError, IndexError):
            continue
        out.append((samples, inst, cur, r[0], r[1].strip()[:90]))
    ts = sum(o[0] for o in out) or 1
    ti = sum(o[1] for o in out) or 1
    print(f"# {path}: {ts} stall samples, {ti} warp instructions")
    print(f"{'samp%':>6} {'inst%':>6}  file:line  source")
    for s, i, f, ln, src in sorted(out, key=lambda o: -o[0])[:top]:
        print(f"{100 * s / ts:6.2f} {100 * i / ti:6.2f}  {f}:{ln}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
