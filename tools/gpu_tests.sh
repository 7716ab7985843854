#!/bin/bash
# GPU parity suite without -x (every failure listed) plus smoke. PYTEST_K
# selects tests by keyword expression (pytest -k).
mkdir -p gpurun_out
if [ -n "$PYTEST_K" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -rf -k "$PYTEST_K" > gpurun_out/pytest_gpu.log 2>&1
else
  timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1
fi
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
exit 0
