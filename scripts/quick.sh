#!/bin/bash
# quick A/B: golden parity (exact64 only) + short C3 bench of the default path
mkdir -p gpurun_out
T=${TAG:-q}
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -p no:cacheprovider -k "exact64 or determin" > gpurun_out/pytest_${T}.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_${T}.log; tail -2 gpurun_out/pytest_${T}.log
timeout 300 python bench.py --steps 32 --warmup 3 --no-cpu-baseline --e2e-steps 2 ${BARGS} > gpurun_out/bench_${T}.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/bench_${T}.log').read().strip().splitlines()[-1]); print('ms/view', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()})" || tail -5 gpurun_out/bench_${T}.log
