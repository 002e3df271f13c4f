#!/bin/bash
mkdir -p gpurun_out
STP_DEBUG_BWD=1 timeout 1500 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -p no:cacheprovider -s 2>&1 | grep -E "stp_backward|passed|failed|FAILED" | tail -20
