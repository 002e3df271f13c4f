#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/sweep_sort.log
for it in ${ITS:-8 12 16}; do
  STP_NVCC_EXTRA="-DSTP_SORT_ITEMS=$it" python paper_2402_00525_b200/build.py --force > /dev/null 2>&1
  timeout 300 python bench.py --steps 16 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print('items $it sort+ranges', round(d['stage_ms']['K4+K5 sort+ranges'],3))" >> gpurun_out/sweep_sort.log
done
cat gpurun_out/sweep_sort.log
