"""Instructions and stall samples per step phase (source-line ranges located by
marker strings in the current sources) from an ncu source page CSV.

  python scripts/ncu_phases.py cs.csv
"""
import collections
import csv
import sys

SRC = "paper_2507_01522_b200/csrc/"
tile = open(SRC + "vy_tile.cuh").read().split("\n")


def find(marker, start=0):
    for i in range(start, len(tile)):
        if marker in tile[i]:
            return i + 1
    raise KeyError(marker)


marks = [
    ("load/issue", "__device__ __forceinline__ void tile_issue("),
    ("envelope/clip/tree fns", "// charge envelope"),
    ("reset/frame/globals", "// reset_env (_kernel.pyx:239-261)"),
    ("stage_port_obs/store_port", "struct ObsSink {"),
    ("phase1 actions", "  // phase 1: apply actions"),
    ("tree excess/fit", "  // tree: excess on the requested currents"),
    ("phase2 charge/depart", "  // phases 2+3: charge"),
    ("battery", "  double e_b = 0.0, bgot = 0.0;"),
    ("arrivals", "  // phase 4: arrivals"),
    ("reward/advance", "  // reward (_kernel.pyx:511-551)"),
    ("obs tail/readout", "// ---- observation"),
]
starts = [(find(m), name) for name, m in marks]
starts.sort()


def phase(fname, line):
    if fname != "vy_tile.cuh":
        return fname
    name = "header"
    for s, n in starts:
        if line >= s:
            name = n
    return name


fname = hdr = None
inst = collections.Counter()
samp = collections.Counter()
for r in csv.reader(open(sys.argv[1])):
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
        p = phase(fname, int(r[0]))
        inst[p] += int(d["Instructions Executed"] or 0)
        samp[p] += int(d["Warp Stall Sampling (All Samples)"] or 0)
    except ValueError:
        pass
ti, ts = sum(inst.values()) or 1, sum(samp.values()) or 1
print(f"{'phase':28s} {'inst%':>6s} {'stall%':>7s}")
for p in sorted(inst, key=lambda p: -samp[p]):
    print(f"{p:28s} {inst[p] / ti * 100:6.1f} {samp[p] / ts * 100:7.1f}")
