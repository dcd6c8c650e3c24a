#!/bin/bash
# DRAM bytes of every k_step launch over one whole 288-step day of the bench
# workload (ncu: dram__bytes_read.sum + dram__bytes_write.sum per launch), to
# compare the kernel's real traffic with the 1414 B/env-step step contract.
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:k_step --launch-skip 5 -c 288 --csv --log-file gpurun_out/day_dram.csv \
    python bench.py --steps 288 --warmup 5 --no-cpu --no-extras > /dev/null 2>&1
python - <<'PY'
import csv, collections, json
rows = [r for r in csv.reader(open("gpurun_out/day_dram.csv")) if len(r) > 10 and r[0].isdigit()]
per = collections.defaultdict(dict)
for r in rows:
    unit, val = r[-2], float(r[-1].replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6}.get(unit, 1)
    per[r[0]][r[-3]] = val * scale
B = 1 << 20
reads = [p["dram__bytes_read.sum"] for p in per.values()]
writes = [p["dram__bytes_write.sum"] for p in per.values()]
out = {"launches": len(per), "bytes_per_env_step_day_avg": (sum(reads) + sum(writes)) / len(per) / B,
       "read_per_env_step": sum(reads) / len(per) / B, "write_per_env_step": sum(writes) / len(per) / B,
       "min_per_env_step": min(r + w for r, w in zip(reads, writes)) / B,
       "max_per_env_step": max(r + w for r, w in zip(reads, writes)) / B}
print(json.dumps(out))
json.dump(out, open("gpurun_out/day_dram.json", "w"), indent=1)
PY
