#!/bin/bash
mkdir -p gpurun_out
T=${TAG:-se}
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider -k "sort_error or globalz or golden_parity" > gpurun_out/pytest_${T}.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_${T}.log; tail -40 gpurun_out/pytest_${T}.log | grep -v "^\.\+ *\[" | tail -30
