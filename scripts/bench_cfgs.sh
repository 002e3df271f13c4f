#!/bin/bash
# short bench of each BASELINE config that fits one GPU (no tests)
mkdir -p gpurun_out
T=${TAG:-cfg}
for c in ${CFGS:-C2 C4 C5}; do
  timeout 600 python bench.py --config $c --steps 16 --warmup 3 --no-cpu-baseline --e2e-steps 4 --views 16 > gpurun_out/bench_${T}_$c.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bench_${T}_$c.log').read().strip().splitlines()[-1]); c=d['config']; print('$c', c['gaussians'], c['width'], c['height'], 'entries', int(c['mean_entries']), 'ms/view', round(d['ms_per_step'],3), 'views/s', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), {k: round(v,3) for k,v in d['stage_ms'].items()})" || tail -5 gpurun_out/bench_${T}_$c.log
done
