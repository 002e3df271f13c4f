#!/bin/bash
mkdir -p gpurun_out
T=${TAG:-bw}
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x --timeout 900 -p no:cacheprovider -k "backward" > gpurun_out/pytest_${T}.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_${T}.log; tail -60 gpurun_out/pytest_${T}.log | grep -v "^\.\+ *\[" | tail -50
