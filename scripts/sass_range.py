"""Print the SASS of one kernel whose line info falls in a source-line range
(nvdisasm -g listing).  python scripts/sass_range.py listing kernel file lo hi"""
import re
import sys

path, kern, fname, lo, hi = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), int(sys.argv[5])
inside, cur, out = False, None, []
for l in open(path):
    if l.startswith("//---------------------"):
        inside = kern in l
        continue
    if not inside:
        continue
    m = re.search(r'File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        out.append((int(m.group(1), 16), cur, m.group(2).strip()))
addrs = [a for a, c, _ in out if c and c[0] == fname and lo <= c[1] < hi]
a0, a1 = min(addrs), max(addrs)
print(f"{(a1 - a0) // 16 + 1} instructions from {a0:x} to {a1:x}")
for a, c, ins in out:
    if a0 <= a <= a1:
        print(f"{a:5x} {c[0][:8]}:{c[1]:<4} {ins[:90]}")
