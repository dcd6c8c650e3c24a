"""Static SASS statistics of one kernel in the built library.

  python scripts/sass_stats.py [kernel-substring] [--ops]
"""
import collections
import re
import subprocess
import sys

name = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "k_step"
lib = "paper_2507_01522_b200/libvoltyard_b200.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
cur, ops = None, collections.Counter()
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    if cur and name in cur:
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m:
            ops[m.group(2)] += 1
print(f"{name}: {sum(ops.values())} SASS instructions")
if "--ops" in sys.argv:
    for op, n in ops.most_common(30):
        print(f"  {op:24s} {n}")
