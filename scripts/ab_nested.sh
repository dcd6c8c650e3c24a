#!/bin/bash
# A/B the C5 station layouts (scripts/probe_nested.py) over variant libraries.
#   bash scripts/ab_nested.sh build/ab/a.so build/ab/b.so ...
LIB=paper_2507_01522_b200/libvoltyard_b200.so
cp $LIB /tmp/_orig.so
for rep in 1 2; do
for v in "$@"; do
  cp "$v" $LIB
  echo "$v rep$rep: $(timeout 300 python scripts/probe_nested.py 2>/dev/null | tail -1)"
done
done
cp /tmp/_orig.so $LIB
