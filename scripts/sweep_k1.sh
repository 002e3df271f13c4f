#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/sweep_k1.log
for v in "2 0" "3 0" "4 0" "3 1" "4 1"; do set -- $v
  STP_NVCC_EXTRA="-DSTP_K1_MINB=$1 -DSTP_SPLIT_SH=$2" python paper_2402_00525_b200/build.py --force > /dev/null 2>&1
  timeout 300 python bench.py --steps 16 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print('k1 minb $1 split $2', round(d['stage_ms']['K0+K1 preprocess'],3))" >> gpurun_out/sweep_k1.log
done
cat gpurun_out/sweep_k1.log
