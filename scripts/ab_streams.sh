#!/bin/bash
mkdir -p gpurun_out
for st in 1 2 3; do
  timeout 300 python bench.py --steps 48 --warmup 4 --no-cpu-baseline --e2e-steps 2 --streams $st > gpurun_out/b_st$st.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/b_st$st.log').read().strip().splitlines()[-1]); print('streams $st', round(d['ms_per_step'],3), 'views/s', round(d['value'],1), {k: round(v,3) for k,v in d['stage_ms'].items()})" || tail -5 gpurun_out/b_st$st.log
done
