#!/bin/bash
./tools/micro/dmma_probe > gpurun_out/dmma_probe.txt 2>&1
for mb in 0 200; do
  echo "== persist $mb MB" >> gpurun_out/sweep2.txt
  PD_L2_PERSIST_MB=$mb bash tools/abia_sweep.sh 4 5 6 >> gpurun_out/sweep2.txt 2>&1
done
