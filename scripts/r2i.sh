#!/bin/bash
O=gpurun_out/r2i; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_reference_replay.py -m gpu -q -rf -k "golden or pixelsort or window or config or full or backward or reference" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python scripts/window_timing.py 0 3 8 24 > $O/win_base.log 2>&1
for v in fullold full32 full128; do STP_LIB_VARIANT=paper_2402_00525_b200/variants/libstp_$v.so timeout 600 python scripts/window_timing.py 0 > $O/win_$v.log 2>&1; done
