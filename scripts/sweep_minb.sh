#!/bin/bash
# launch-bounds sweep of both K6 kernels on C3 (bench, 24 steps each)
mkdir -p gpurun_out; : > gpurun_out/sweep_minb.log
for mb in ${MBS:-4 5 6}; do
  STP_NVCC_EXTRA="-DSTP_EXACT_MINB=$mb -DSTP_FAST_MINB=$mb" python paper_2402_00525_b200/build.py --force > /dev/null 2>&1
  for ex in "" "--fast32"; do
    timeout 300 python bench.py --steps 24 --warmup 3 --no-cpu-baseline --e2e-steps 2 $ex > gpurun_out/b.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print('minb $mb $ex', round(d['stage_ms']['K6 render'],3), 'resolves', d['config']['mean_resolves'], 'fb', d['config']['mean_exact_items'])" >> gpurun_out/sweep_minb.log 2>&1 || tail -3 gpurun_out/b.log >> gpurun_out/sweep_minb.log
  done
done
cat gpurun_out/sweep_minb.log
