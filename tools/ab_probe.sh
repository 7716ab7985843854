#!/bin/bash
# A/B kernel timing: for each library variant in paper_1609_06779_b200/lib/ab/*.so
# (alternating, ROUNDS times) run tools/route_probe.py on each workload.
# Usage: ROUNDS=2 tools/ab_probe.sh "c2j c5j" variantA variantB ...
L=paper_1609_06779_b200/lib
wls=$1; shift
cp $L/libpardyn_b200.so /tmp/pd_keep.so
for r in $(seq ${ROUNDS:-2}); do
  for v in "$@"; do
    cp $L/ab/$v.so $L/libpardyn_b200.so
    for c in $wls; do echo "$v $(timeout 120 python tools/route_probe.py $c 0 2>&1 | tail -1)"; done
  done
done
cp /tmp/pd_keep.so $L/libpardyn_b200.so
