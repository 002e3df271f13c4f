#!/bin/bash
# GlobalZ vs Hierarchical on the same configs (the paper's A/B)
mkdir -p gpurun_out
for c in ${CFGS:-C3}; do for m in ${MODES:-globalz hierarchical}; do
  timeout 600 python bench.py --config $c --mode $m --steps 32 --warmup 4 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_${TAG:-gzb}_${c}_${m//:/_}.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bench_${TAG:-gzb}_${c}_${m//:/_}.log').read().strip().splitlines()[-1]); c=d['config']; print('$c $m entries', int(c['mean_entries']), 'ms/view', round(d['ms_per_step'],3), 'views/s', round(d['value'],1), {k: round(v,3) for k,v in d['stage_ms'].items()})" || tail -5 gpurun_out/bench_${TAG:-gzb}_${c}_${m//:/_}.log
done; done
