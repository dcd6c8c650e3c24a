#!/bin/bash
# Time the bench's main leg (day-window k_step) with each variant library in turn.
#   bash scripts/ab_run.sh build/ab/a.so build/ab/b.so ...
LIB=paper_2507_01522_b200/libvoltyard_b200.so
cp $LIB /tmp/_orig.so
for rep in 1 2; do
for v in "$@"; do
  cp "$v" $LIB
  r=$(timeout 300 python bench.py --no-cpu --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['roofline']['kernel_ms'],4), round(d['value']/1e9,3))")
  echo "$v rep$rep kernel_ms/value(e9): $r"
done
done
cp /tmp/_orig.so $LIB
