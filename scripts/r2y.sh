#!/bin/bash
# bench A/B of the e2e copy stream and views in flight
O=gpurun_out/${TAG:-r2y}; mkdir -p $O
for st in 2 3 2; do
  timeout 300 python bench.py --steps 64 --warmup 5 --no-cpu-baseline --e2e-steps 32 --streams $st > $O/bench_s$st.json 2>$O/bench_s$st.err
  python -c "import json; d=json.loads(open('$O/bench_s$st.json').read().strip().splitlines()[-1]); print('streams $st', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), round(d['ms_per_step'],4))" >> $O/summary.txt 2>&1
done
cat $O/summary.txt
