#!/bin/bash
# Fast iteration on the GPU box: parity tests, short bench, K6 phase profile.
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py -q -x --timeout 200 -p no:cacheprovider > gpurun_out/iter_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/iter_pytest.log
timeout 300 python bench.py --steps 32 --warmup 3 --no-cpu-baseline --e2e-steps 4 > gpurun_out/iter_bench.log 2>&1
STP_NVCC_EXTRA=-DSTP_PHASE_PROF python paper_2402_00525_b200/build.py --force > /dev/null 2>&1
timeout 200 python scripts/phase_prof.py C3 2>/dev/null > gpurun_out/iter_prof.log
tail -2 gpurun_out/iter_pytest.log
python -c "import json; d=json.loads(open('gpurun_out/iter_bench.log').read().strip().splitlines()[-1]); print('ms/view', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, 'e2e', round(d['e2e']['value'],1))"
cat gpurun_out/iter_prof.log
