#!/bin/bash
# A/B pass: alternate lib/ab/old.so and lib/ab/new.so on the given workloads
# (tools/ab_probe.sh), then the GPU tests matching a keyword on the new build.
# Usage: tools/ab_run.sh "c2 c5a" "abia or ABIA"
mkdir -p gpurun_out
ROUNDS=${ROUNDS:-3} bash tools/ab_probe.sh "$1" old new > gpurun_out/ab.txt 2>&1
cp paper_1609_06779_b200/lib/ab/new.so paper_1609_06779_b200/lib/libpardyn_b200.so
timeout 900 python -m pytest tests -m gpu -q -x -k "$2" > gpurun_out/pytest_ab.log 2>&1; echo "exit $?" >> gpurun_out/pytest_ab.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ab.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_ab.log
