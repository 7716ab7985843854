#!/bin/bash
# A/B the ABIA TMA kernel variants (PD_ABIA_VARIANT) on c2; one JSON line each.
for v in "$@"; do
  PD_ABIA_VARIANT=$v timeout 300 python bench.py --workload ${WL:-c2} --steps ${STEPS:-1000} --warmup 100 --no-extra --no-cpu --no-e2e 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('variant $v', round(d['ms_per_step']*1000,1), 'us/step', round(d['value']/1e6,1), 'M solves/s', 'hbm_frac', round(d['roofline']['frac'],3), d['clocks'])"
done
