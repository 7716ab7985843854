#!/bin/bash
# Quick GPU pass after a kernel change: GPU parity suite, c2 bench line (no CPU
# leg), a few workload lines, and DRAM bytes of the top ABIA launch.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 500 --warmup 50 --no-cpu --no-e2e > gpurun_out/quick.json 2>gpurun_out/quick.err
for w in ${WLS:-c5a c3 c2j}; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-extra --no-cpu --no-e2e >> gpurun_out/quick.json 2>>gpurun_out/quick.err
done
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active -k regex:abia -s 3 -c 1 \
  python bench.py --steps 2 --warmup 3 --no-extra --no-cpu --no-e2e > gpurun_out/quick_ncu.txt 2>&1
exit 0
