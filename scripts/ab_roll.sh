#!/bin/bash
# A/B variant libraries on the bench's main leg (20-step mid-day window, whole
# day) and the fused rollout (mid-day probe): bash scripts/ab_lib.sh a.so b.so ...
LIB=paper_2507_01522_b200/libvoltyard_b200.so
cp $LIB /tmp/_orig.so
for rep in 1 2; do
for v in "$@"; do
  cp "$v" $LIB
  r=$(timeout 300 python bench.py --no-cpu --no-extras --steps 20 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['roofline']['kernel_ms'],4), round(d['value']/1e9,3))")
  d=$(timeout 300 python bench.py --no-cpu --no-extras --steps 288 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['roofline']['kernel_ms'],4), round(d['value']/1e9,3))")
  o=$(timeout 300 python scripts/probe_rollout.py 2>/dev/null | tail -1)
  echo "$v rep$rep window20: $r   day288: $d   $o"
done
done
cp /tmp/_orig.so $LIB
