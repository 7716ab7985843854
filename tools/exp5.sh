#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/exp5_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/exp5_pytest.txt
timeout 600 python bench.py --no-extra > gpurun_out/exp5_bench.json 2> gpurun_out/exp5_bench.err
for v in 10 12; do
  PD_ABIA_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "abia or c1 or pendulum or errors or determin" 2>&1 | tail -1 | sed "s/^/v$v parity: /" >> gpurun_out/exp5.txt
done
