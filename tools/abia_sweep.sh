#!/bin/bash
# A/B ABIA TMA variants on c2: bench timing (no profiler) + DRAM bytes (ncu metrics pass).
mkdir -p gpurun_out
WL=${WL:-c2}
for v in "$@"; do
  PD_ABIA_VARIANT=$v timeout 300 python bench.py --workload $WL --steps 500 --warmup 50 --no-extra --no-cpu --no-e2e 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('variant $v', round(d['ms_per_step']*1000,1), 'us/step', 'hbm_frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
  PD_ABIA_VARIANT=$v timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:abia -s 3 -c 1 \
    python bench.py --workload $WL --steps 2 --warmup 3 --no-extra --no-cpu --no-e2e 2>/dev/null | grep -E "dram__bytes|gpu__time|hit_rate" | sed "s/^/  v$v /"
done
