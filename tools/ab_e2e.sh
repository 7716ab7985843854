#!/bin/bash
# e2e (host-buffer path) A/B: alternate the library variants in lib/ab/ and
# print the bench line's e2e and device values for each.
# Usage: ROUNDS=3 tools/ab_e2e.sh old variantA ...
L=paper_1609_06779_b200/lib
cp $L/libpardyn_b200.so /tmp/pd_keep.so
for r in $(seq ${ROUNDS:-3}); do
  for v in "$@"; do
    cp $L/ab/$v.so $L/libpardyn_b200.so
    timeout 300 python bench.py --steps 200 --warmup 20 --no-extra --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('$v', 'e2e %.2f M/s' % (d['e2e']['value']/1e6), 'device %.1f M/s' % (d['value']/1e6))"
  done
done
cp /tmp/pd_keep.so $L/libpardyn_b200.so
