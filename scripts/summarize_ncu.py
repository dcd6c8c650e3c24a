"""Summarise ncu captures into profiles/ (run here; the .ncu-rep comes back from gpurun).

  python scripts/summarize_ncu.py full  <report.ncu-rep> <out.txt> [--traffic-json profiles/step_kernel_dram_bytes.json]
  python scripts/summarize_ncu.py launches <launches.csv> <out.txt>
"""

from __future__ import annotations

import csv
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("smsp__inst_executed.sum", "instructions executed (warp)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__block_size", "block size"),
    ("launch__grid_size", "grid size"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("launch__occupancy_limit_shared_mem", "CTA limit by smem"),
    ("launch__occupancy_limit_registers", "CTA limit by registers"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe active %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
]


def raw_metrics(rep: str) -> list[dict]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        d["_units"] = dict(zip(hdr, units))
        res.append(d)
    return res


def to_bytes(val: str, unit: str) -> float:
    v = float(val)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return v * scale


def full(rep: str, out: str, traffic_json: str | None) -> None:
    lines = [f"# ncu --set full summary of {rep}", ""]
    for d in raw_metrics(rep):
        name = d.get("Kernel Name", "?")
        lines.append(f"## {name}")
        u = d["_units"]
        for k, label in KEYS:
            if k in d:
                lines.append(f"  {label:34s} {d[k]} {u.get(k, '')}")
        stalls = sorted(((k, float(v)) for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled_")
                         and k.endswith("_per_issue_active.ratio") and v not in ("", "n/a")), key=lambda kv: -kv[1])
        lines.append("  stall cycles per issued instruction: " + ", ".join(
            f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={v:.2f}"
            for k, v in stalls[:8]))
        rd = to_bytes(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"])
        wr = to_bytes(d["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
        lines.append(f"  DRAM bytes per launch (read + write): {rd + wr:.0f}")
        if traffic_json and "k_step" in name:
            with open(traffic_json, "w") as fh:
                json.dump({"kernel": name, "bytes_per_launch": rd + wr, "read": rd, "write": wr, "source": rep}, fh,
                          indent=1)
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def launches(path: str, out: str) -> None:
    rows = [r for r in csv.reader(line for line in open(path) if not line.startswith("=="))]
    hdr = rows[0]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[1:]:
        agg[r[ik].split("(")[0]].append(float(r[iv]))
    tot = sum(sum(v) for v in agg.values())
    lines = [f"# launch list (ncu gpu__time_duration.sum, cold-cache, serialised) from {path}", "",
             f"{'kernel':60s} {'launches':>8s} {'mean us':>10s} {'share':>7s}"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{k[:60]:60s} {len(v):8d} {sum(v) / len(v) / 1e3:10.1f} {sum(v) / tot * 100:6.1f}%")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "full":
        tj = sys.argv[sys.argv.index("--traffic-json") + 1] if "--traffic-json" in sys.argv else None
        full(sys.argv[2], sys.argv[3], tj)
    else:
        launches(sys.argv[2], sys.argv[3])
