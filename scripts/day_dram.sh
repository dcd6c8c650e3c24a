#!/bin/bash
# DRAM bytes of every k_step launch over one whole 288-step day of the bench
# workload (ncu: dram__bytes_read.sum + dram__bytes_write.sum per launch), indexed
# by step of the day, so bench.py can report the measured traffic of whatever
# window it times (roofline.traffic).  Output: gpurun_out/day_dram.json
# (copy to profiles/r2_k_step_day_dram.json).
W=5
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:k_step --launch-skip $W -c 288 --csv --log-file gpurun_out/day_dram.csv \
    python bench.py --steps 288 --warmup $W --no-cpu --no-extras > /dev/null 2>&1
W=$W python - <<'PY'
import csv, collections, json, os
W = int(os.environ["W"])
rows = [r for r in csv.reader(open("gpurun_out/day_dram.csv")) if len(r) > 10 and r[0].isdigit()]
per = collections.defaultdict(dict)
for r in rows:
    unit, val = r[-2], float(r[-1].replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6}.get(unit, 1)
    per[int(r[0])][r[-3]] = val * scale
B = 1 << 20
ids = sorted(per)
by_step = [0.0] * 288
dur = [0.0] * 288
for i, lid in enumerate(ids):
    p = per[lid]
    by_step[(W + i) % 288] = p["dram__bytes_read.sum"] + p["dram__bytes_write.sum"]
    dur[(W + i) % 288] = p["gpu__time_duration.sum"]
reads = [per[i]["dram__bytes_read.sum"] for i in ids]
writes = [per[i]["dram__bytes_write.sum"] for i in ids]
out = {"launches": len(ids), "envs": B, "kernel": "vy::k_step<1> via vy_step_random (fused RandomPolicy)",
       "how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none "
              "-k regex:k_step --launch-skip 5 -c 288 python bench.py --steps 288 --warmup 5 --no-cpu --no-extras",
       "bytes_per_env_step_day_avg": (sum(reads) + sum(writes)) / len(ids) / B,
       "read_per_env_step": sum(reads) / len(ids) / B, "write_per_env_step": sum(writes) / len(ids) / B,
       "min_per_env_step": min(by_step) / B, "max_per_env_step": max(by_step) / B,
       "bytes_per_launch_by_step": by_step, "ncu_ns_by_step": dur}
print(json.dumps({k: v for k, v in out.items() if not k.endswith("_by_step")}))
json.dump(out, open("gpurun_out/day_dram.json", "w"), indent=1)
PY
