#!/bin/bash
# A/B the bench's main leg (fused policy step over the driver's 20-step mid-day
# window and a whole day) across variant libraries: bash scripts/ab_window.sh a.so b.so ...
LIB=paper_2507_01522_b200/libvoltyard_b200.so
cp $LIB /tmp/_orig.so
for rep in 1 2 3; do
for v in "$@"; do
  cp "$v" $LIB
  r=$(timeout 300 python bench.py --no-cpu --no-extras --steps 20 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['roofline']['kernel_ms'],4), round(d['value']/1e9,3))")
  d=$(timeout 300 python bench.py --no-cpu --no-extras --steps 288 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['roofline']['kernel_ms'],4), round(d['value']/1e9,3))")
  echo "$v rep$rep window20 kernel_ms/value(e9): $r   day288: $d"
done
done
cp /tmp/_orig.so $LIB
