#!/bin/bash
# Alternate several library variants in lib/ab/ (tools/route_probe.py per workload).
# Usage: ROUNDS=3 tools/ab_multi.sh "c2 c5a" old v1 v2 ...
L=paper_1609_06779_b200/lib
wls=$1; shift
cp $L/libpardyn_b200.so /tmp/pd_keep.so
for r in $(seq ${ROUNDS:-3}); do
  for v in "$@"; do
    cp $L/ab/$v.so $L/libpardyn_b200.so
    for c in $wls; do echo "$v $(timeout 120 python tools/route_probe.py $c 0 2>&1 | tail -1 | cut -c1-40)"; done
  done
done
cp /tmp/pd_keep.so $L/libpardyn_b200.so
