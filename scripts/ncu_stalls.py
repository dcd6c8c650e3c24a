"""Stall reasons per CUDA source line from an ncu source page (cuda,sass CSV).

  python scripts/ncu_stalls.py cs.csv [reason ...]   (reasons: short_sb wait no_inst long_sb ...)
"""
import collections
import csv
import sys

path = sys.argv[1]
reasons = sys.argv[2:] or ["short_sb", "wait", "no_inst", "long_sb"]
fname = hdr = None
agg = {r: collections.Counter() for r in reasons}
for r in csv.reader(open(path)):
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
    key = f"{fname}:{r[0]} {r[1].strip()[:60]}"
    for k in reasons:
        try:
            agg[k][key] += int(d.get("stall_" + k) or 0)
        except ValueError:
            pass
for k, a in agg.items():
    t = sum(a.values()) or 1
    print(f"== {k} {t}")
    for key, v in a.most_common(14):
        print(f"  {v / t * 100:5.1f}% {key}")
