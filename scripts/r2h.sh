#!/bin/bash
O=gpurun_out/r2h; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -k "golden or pixelsort or window or config" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python scripts/window_timing.py > $O/win_base.log 2>&1
STP_LIB_VARIANT=paper_2402_00525_b200/variants/libstp_heap1.so timeout 600 python scripts/window_timing.py 3 4 8 > $O/win_heap1.log 2>&1
