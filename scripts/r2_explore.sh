#!/bin/bash
O=gpurun_out/${1:-r2b}
mkdir -p $O
timeout 900 python -m pytest tests/test_fullsize_parity.py tests/test_gpu_parity.py -m gpu -q -rs -k "fullsize or window or pixelsort or config_errors" > $O/pytest_sel.log 2>&1; echo "rc=$?" >> $O/pytest_sel.log
bash scripts/replay_ref.sh $O/replay
echo done
