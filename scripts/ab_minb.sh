#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/ab_minb.log
for mb in 4 5; do
  STP_NVCC_EXTRA="-DSTP_EXACT_MINB=$mb" python paper_2402_00525_b200/build.py --force > /dev/null 2>&1
  timeout 300 python bench.py --steps 32 --warmup 3 --no-cpu-baseline --e2e-steps 2 --streams 1 > gpurun_out/b.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print('minb $mb K6', round(d['stage_ms']['K6 render'],3))" >> gpurun_out/ab_minb.log
done
cat gpurun_out/ab_minb.log
python paper_2402_00525_b200/build.py --force > /dev/null 2>&1
