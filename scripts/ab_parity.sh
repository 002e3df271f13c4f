#!/bin/bash
# Parity subset on the default build, then an A/B of knob variants (built
# here first with build.py --variant TAG -DKNOB=..).
# Usage: TAG=x AB_VARIANTS="v1 v2" bash scripts/ab_parity.sh
O=gpurun_out/${TAG:-ab}; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_parity.py -m gpu -q -rf -x \
  -k "golden or c1 or c3_layout or fullsize_c2 or fullsize_c3 or c4_law or elongated or batch" > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
[ -z "$TAIL_PROF" ] || STP_LIB_VARIANT=paper_2402_00525_b200/variants/libstp_tailp.so \
  timeout 300 python scripts/tail_prof.py C3 > $O/tail.json 2>&1
bash scripts/ab.sh ${TAG:-ab}_ab ${AB_VARIANTS}
