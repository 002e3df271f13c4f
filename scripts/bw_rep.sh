#!/bin/bash
mkdir -p gpurun_out
for i in 1 2 3; do
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider -k "backward_oracle" 2>&1 | tail -1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -p no:cacheprovider -k "backward or sort_error or pixelsort" 2>&1 | tail -3
