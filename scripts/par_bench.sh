#!/bin/bash
# whole parity file + 2 benches
mkdir -p gpurun_out
T=${TAG:-pb}
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_${T}.log 2>&1
echo "pytest exit $?"; tail -2 gpurun_out/pytest_${T}.log | head -1
REPS=2 bash scripts/bench3.sh
