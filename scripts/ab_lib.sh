#!/bin/bash
# A/B the step kernel across alternative builds of the library (tuning aid).
for lib in paper_2507_01522_b200/libvoltyard_b200.so "$@"; do
  cp paper_2507_01522_b200/libvoltyard_b200.so /tmp/_orig.so 2>/dev/null
  if [ "$lib" != paper_2507_01522_b200/libvoltyard_b200.so ]; then cp "$lib" paper_2507_01522_b200/libvoltyard_b200.so; fi
  echo "== $lib"; timeout 300 python scripts/probe_step.py 2>&1 | head -1
  cp /tmp/_orig.so paper_2507_01522_b200/libvoltyard_b200.so
done
