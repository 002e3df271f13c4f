#!/bin/bash
O=gpurun_out/r2o; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_parity.py -m gpu -q -rf -x -k "golden or c1 or c3_layout or fullsize_c3 or queues or records or backward" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
bash scripts/ab.sh r2o_ab prefast
