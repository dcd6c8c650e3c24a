#!/bin/bash
# k_step day-window time vs warps per CTA (resident warps per SM = CTAs/SM x warps).
for w in 8 4 5 3 2 1; do
  r=$(VY_WARPS_PER_CTA=$w timeout 300 python bench.py --no-cpu --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['roofline']['kernel_ms'],4), round(d['value']/1e9,3))")
  echo "warps/CTA $w: kernel_ms/value(e9): $r"
done
