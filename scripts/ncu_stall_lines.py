"""Warp-stall samples and executed instructions of one kernel by source line
and by SASS opcode, from an ncu source-page export (SASS view) joined with the
nvdisasm -g line table of the same library build.

  ncu -i rep.ncu-rep --page source --csv --print-source sass > k.csv
  python scripts/ncu_stall_lines.py k.csv _ZN2vy6k_stepILi1EEEvNS_6ParamsE [vy_abi]
"""
import collections
import csv
import glob
import os
import re
import subprocess
import sys
import tempfile

csv_path, mangled = sys.argv[1], sys.argv[2]
unit = sys.argv[3] if len(sys.argv) > 3 else "vy_abi"
lib = os.path.abspath("paper_2507_01522_b200/libvoltyard_b200.so")
with tempfile.TemporaryDirectory() as tmp:
    subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, capture_output=True, check=True)
    cubin = [c for c in glob.glob(os.path.join(tmp, "*.cubin")) if unit in c][0]
    listing = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.splitlines()
inside, cur, off2line = False, None, {}
for line in listing:
    if line.startswith("//-----"):
        inside = mangled in line
        continue
    if not inside:
        continue
    m = re.search(r'File "([^"]+)", line (\d+)', line)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        off2line[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(csv_path)))
hdr, data = rows[1], rows[2:]
ia, isrc = hdr.index("Address"), hdr.index("Source")
isamp, iex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
base = int(data[0][ia], 16)
byline = collections.defaultdict(lambda: [0, 0, collections.Counter()])
byop, byop_s = collections.Counter(), collections.Counter()
tot_s = tot_e = 0
for r in data:
    s, e = int(r[isamp] or 0), int(r[iex] or 0)
    b = byline[off2line.get(int(r[ia], 16) - base)]
    b[0] += s
    b[1] += e
    for i in stall_cols:
        if r[i] and int(r[i]):
            b[2][hdr[i][6:]] += int(r[i])
    toks = r[isrc].split()
    op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
    byop[op] += e
    byop_s[op] += s
    tot_s += s
    tot_e += e
print(f"{mangled}: {tot_s} stall samples, {tot_e} warp instructions executed")
print("\n# top source lines by stall samples (share of samples, share of executed instructions, top stall reasons)")
for ln, (s, e, c) in sorted(byline.items(), key=lambda kv: -kv[1][0])[:40]:
    print(f"{str(ln):34s} samples {100 * s / tot_s:5.1f}%  inst {100 * e / tot_e:5.1f}%   "
          + " ".join(f"{k}={v}" for k, v in c.most_common(3)))
print("\n# executed instructions by opcode")
for op, e in byop.most_common(25):
    print(f"{op:10s} inst {100 * e / tot_e:5.1f}%  samples {100 * byop_s[op] / tot_s:5.1f}%")
