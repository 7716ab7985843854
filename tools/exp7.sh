#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/exp7_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/exp7_pytest.txt
for v in 10 12 13 14; do
  PD_ABIA_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "abia or c1 or pendulum or errors or determin or chunked" 2>&1 | tail -1 | sed "s/^/v$v parity: /" >> gpurun_out/exp7.txt
done
for v in 4 12 13 14 10; do
  PD_ABIA_VARIANT=$v timeout 300 python bench.py --workload c2 --steps 300 --warmup 30 --no-extra --no-cpu --no-e2e 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('abia c2 variant $v', round(d['ms_per_step']*1000,1), 'us/step', 'hbm_frac', round(d['roofline']['frac'],3))" >> gpurun_out/exp7.txt 2>&1
done
for v in 4 12 13; do
  PD_ABIA_VARIANT=$v timeout 300 python bench.py --workload c5a --steps 10 --warmup 3 --no-extra --no-cpu --no-e2e 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('abia c5a variant $v', round(d['ms_per_step'],3), 'ms/step', 'hbm_frac', round(d['roofline']['frac'],3))" >> gpurun_out/exp7.txt 2>&1
done
for w in c2j c5j; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-extra --no-cpu --no-e2e 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', round(d['ms_per_step'],3), 'ms/step', 'fp64_frac', round(d['roofline_fp64']['frac'],3))" >> gpurun_out/exp7.txt 2>&1
done
for c in 1 4 8; do PD_E2E_CHUNKS=$c timeout 300 python tools/e2e_probe.py >> gpurun_out/exp7.txt 2>&1; done
