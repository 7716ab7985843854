#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/exp6_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/exp6_pytest.txt
timeout 900 python bench.py > gpurun_out/exp6_bench.json 2> gpurun_out/exp6_bench.err
for w in c5a c5j c5c; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-extra --no-cpu --no-e2e >> gpurun_out/exp6_wl.jsonl 2>> gpurun_out/exp6_bench.err
done
PD_ABIA_VARIANT=4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:abia -s 3 -c 1 -o gpurun_out/ncu_c2_v4f python bench.py --workload c2 --steps 2 --warmup 3 --no-extra --no-cpu --no-e2e > /dev/null 2>&1
PD_ABIA_VARIANT=12 timeout 600 ncu --set full --clock-control none --import-source on -k regex:abia -s 3 -c 1 -o gpurun_out/ncu_c2_v12 python bench.py --workload c2 --steps 2 --warmup 3 --no-extra --no-cpu --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:jsiia_dmma -s 3 -c 1 -o gpurun_out/ncu_c2j_dmma python bench.py --workload c2j --steps 2 --warmup 3 --no-extra --no-cpu --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:jsiia_dmma -s 3 -c 1 -o gpurun_out/ncu_c5j_dmma python bench.py --workload c5j --steps 2 --warmup 3 --no-extra --no-cpu --no-e2e > /dev/null 2>&1
exit 0
