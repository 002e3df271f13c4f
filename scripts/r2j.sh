#!/bin/bash
O=gpurun_out/r2j; mkdir -p $O
for v in full16 full24 full48; do STP_LIB_VARIANT=paper_2402_00525_b200/variants/libstp_$v.so timeout 600 python scripts/window_timing.py 0 > $O/win_$v.log 2>&1; done
timeout 600 python scripts/window_timing.py 0 > $O/win_full32.log 2>&1
