#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/sweep.log
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x --timeout 200 -p no:cacheprovider > gpurun_out/sweep_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/sweep_pytest.log
for mb in ${MBS:-4 5}; do
  sed -i "s/__launch_bounds__(kRenderThreads, [0-9])/__launch_bounds__(kRenderThreads, $mb)/" paper_2402_00525_b200/csrc/stp_render.cu
  python paper_2402_00525_b200/build.py --force > /dev/null 2>&1
  echo "== minblocks $mb" >> gpurun_out/sweep.log
  timeout 300 python bench.py --steps 32 --warmup 3 --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()})" >> gpurun_out/sweep.log 2>&1
  STP_NVCC_EXTRA=-DSTP_PHASE_PROF python paper_2402_00525_b200/build.py --force > /dev/null 2>&1
  timeout 200 python scripts/phase_prof.py C3 2>/dev/null >> gpurun_out/sweep.log
done
tail -2 gpurun_out/sweep_pytest.log; cat gpurun_out/sweep.log
