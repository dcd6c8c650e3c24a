"""Static SASS instruction count per source line range of one kernel
(nvdisasm -g of the library's cubin).  Tuning aid for code size.

  python scripts/sass_lines.py <sass-with-lineinfo> <kernel-mangled-substring>
"""
import collections
import re
import sys

path, kern = sys.argv[1], sys.argv[2]
cnt = collections.Counter()
inside = False
cur = None
for line in open(path):
    if line.startswith("//---------------------"):
        inside = kern in line
        continue
    if not inside:
        continue
    m = re.search(r'File "([^"]+)", line (\d+)', line)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", line) and cur:
        cnt[cur] += 1
tot = sum(cnt.values())
print("total", tot)
byfile = collections.Counter()
for (f, l), v in cnt.items():
    byfile[f] += v
print(byfile)
for (f, l), v in sorted(cnt.items(), key=lambda x: -x[1])[:40]:
    print(f"{v:5d} {f}:{l}")
