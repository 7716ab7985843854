#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py (every default kernel once, small sizes).
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 30 --error-exitcode 9 python tools/sanitize_run.py \
    > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "$tool exit $?" >> gpurun_out/sanitizer_status.txt
done
exit 0
