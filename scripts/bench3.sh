#!/bin/bash
# bench repeatability: REPS short C3 benches
mkdir -p gpurun_out
for r in $(seq ${REPS:-3}); do
  timeout 300 python bench.py --steps 64 --warmup 5 --no-cpu-baseline --e2e-steps 2 ${BARGS} > gpurun_out/bench_rep.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bench_rep.log').read().strip().splitlines()[-1]); print('ms/view', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()})"
done
