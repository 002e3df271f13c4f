#!/bin/bash
# parity (exact64 + 4K C4-law + elongated rows) and C3 / C4 benches
mkdir -p gpurun_out
T=${TAG:-cc}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider -k "exact64 or determin or c4_law or elongated" > gpurun_out/pytest_${T}.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_${T}.log; tail -3 gpurun_out/pytest_${T}.log
for c in C3 C4; do
  timeout 600 python bench.py --config $c --steps 16 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_${T}_$c.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bench_${T}_$c.log').read().strip().splitlines()[-1]); c=d['config']; print('$c', 'entries', int(c['mean_entries']), 'ms/view', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()})" || tail -5 gpurun_out/bench_${T}_$c.log
done
