"""Top SASS instructions by stall samples with their dominant stall reasons.

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python scripts/ncu_sass_stalls.py src.csv [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], encoding="latin-1")))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = next(r for r in rows if r and r[0] == "Line No")
col = {c: i for i, c in enumerate(hdr)}
stall_cols = [(i, c) for i, c in enumerate(hdr) if c.startswith("stall_") and "Not Issued" not in c]
out = []
for r in rows:
    if len(r) < len(hdr) or not r[2].startswith("0x"):
        continue
    try:
        samp = float(r[col["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    reasons = sorted(((float(r[i] or 0), c[6:]) for i, c in stall_cols), reverse=True)[:3]
    out.append((samp, r[2][-5:], r[3][:60], ", ".join(f"{n}={v:.0f}" for v, n in reasons if v > 0)))
tot = sum(o[0] for o in out) or 1
for samp, addr, sass, rs in sorted(out, reverse=True)[:top]:
    print(f"{100 * samp / tot:5.2f}%  {addr}  {sass:60s}  {rs}")
