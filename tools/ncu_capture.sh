#!/bin/bash
# ncu --set full captures of the top kernel of each workload (1 GPU, one
# launch each after warm-up). Usage: tools/ncu_capture.sh TAG [workload:regex ...]
TAG=$1; shift
mkdir -p gpurun_out
for spec in "$@"; do
  wl=${spec%%:*}; rx=${spec#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s 3 -c 1 \
    -o gpurun_out/ncu_${wl}_${TAG} python bench.py --workload $wl --steps 2 --warmup 3 --no-extra --no-cpu --no-e2e \
    > gpurun_out/ncu_${wl}_${TAG}.log 2>&1
  echo "$spec exit $?" >> gpurun_out/ncu_${TAG}.status
done
exit 0
