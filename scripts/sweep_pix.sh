#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/sweep_pix.log
for u in ${US:-2 3 4}; do
  STP_NVCC_EXTRA="-DSTP_PIX_UNROLL=$u" python paper_2402_00525_b200/build.py --force > /dev/null 2>&1
  timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "exact64 and (c1 or cloud300 or scaled)" -p no:cacheprovider > gpurun_out/pt.log 2>&1; echo "unroll $u pytest $?" >> gpurun_out/sweep_pix.log
  timeout 300 python bench.py --steps 16 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print('unroll $u K6', round(d['stage_ms']['K6 render'],3))" >> gpurun_out/sweep_pix.log
done
cat gpurun_out/sweep_pix.log
