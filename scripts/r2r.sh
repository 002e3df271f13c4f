#!/bin/bash
O=gpurun_out/${TAG:-r2r}; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_parity.py -m gpu -q -rf -x -k "golden or c1 or c3_layout or fullsize_c2 or fullsize_c3 or c4_law or elongated or batch" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
bash scripts/ab.sh ${AB_TAG:-r2r_ab} ${AB_VARIANTS:-k1old}
