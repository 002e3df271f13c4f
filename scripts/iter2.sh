#!/bin/bash
# Fast iteration: parity tests (fast + exact64), short bench of both K6 paths.
mkdir -p gpurun_out
T=${TAG:-it}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 400 -p no:cacheprovider ${PYARGS} > gpurun_out/pytest_${T}.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_${T}.log
tail -15 gpurun_out/pytest_${T}.log
for ex in "" "--fast32"; do
timeout 300 python bench.py --steps 32 --warmup 3 --no-cpu-baseline --e2e-steps 4 $ex > gpurun_out/bench_${T}${ex}.log 2>&1
python -c "import json,sys; d=json.loads(open('gpurun_out/bench_${T}${ex}.log').read().strip().splitlines()[-1]); print('$ex', 'ms/view', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, 'exact_items', d['config'].get('mean_exact_items'), 'resolves', d['config'].get('mean_resolves'))" || tail -20 gpurun_out/bench_${T}${ex}.log
done
