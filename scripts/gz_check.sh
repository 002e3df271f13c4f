#!/bin/bash
# GlobalZ parity (golden + oracle) and the whole parity file
mkdir -p gpurun_out
T=${TAG:-gz}
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_${T}.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_${T}.log; tail -30 gpurun_out/pytest_${T}.log | grep -v "^\.\+ *\[" | tail -25
