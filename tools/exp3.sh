#!/bin/bash
mkdir -p gpurun_out
for v in 10 12 13 14 15; do
  PD_ABIA_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "abia or ABIA or c1 or pendulum or errors or determin" 2>&1 | tail -2 | sed "s/^/v$v parity: /" >> gpurun_out/exp3.txt
done
bash tools/abia_sweep.sh 10 11 12 13 14 15 >> gpurun_out/exp3.txt 2>&1
WL=c5a bash tools/abia_sweep.sh 10 13 >> gpurun_out/exp3.txt 2>&1
