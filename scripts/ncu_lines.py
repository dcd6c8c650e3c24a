"""Aggregate an ncu source page (cuda,sass CSV) per CUDA source line.

  ncu -i rep --page source --csv --print-source cuda,sass > cs.csv
  python scripts/ncu_lines.py cs.csv [top]
"""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows, fname, hdr = [], None, None
with open(path) as f:
    for r in csv.reader(f):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] in ("", "Function Name"):
            continue
        d = dict(zip(hdr, r))
        try:
            inst = int(d["Instructions Executed"] or 0)
            samp = int(d["Warp Stall Sampling (All Samples)"] or 0)
        except ValueError:
            continue
        rows.append((fname, int(r[0]), r[1].strip()[:70], inst, samp))
ti = sum(x[3] for x in rows) or 1
ts = sum(x[4] for x in rows) or 1
print(f"total warp inst {ti}  samples {ts}")
print("== by stall samples")
for x in sorted(rows, key=lambda x: -x[4])[:top]:
    print(f"{x[4] / ts * 100:5.1f}% samp {x[3] / ti * 100:5.1f}% inst  {x[0]}:{x[1]}  {x[2]}")
print("== by instructions executed")
for x in sorted(rows, key=lambda x: -x[3])[:top]:
    print(f"{x[3] / ti * 100:5.1f}% inst {x[4] / ts * 100:5.1f}% samp  {x[0]}:{x[1]}  {x[2]}")
