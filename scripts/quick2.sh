#!/bin/bash
# quick A/B: all GPU parity tests + short C3 bench + launch list
mkdir -p gpurun_out
T=${TAG:-q}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 400 -p no:cacheprovider > gpurun_out/pytest_${T}.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_${T}.log; tail -4 gpurun_out/pytest_${T}.log
timeout 300 python bench.py --steps 32 --warmup 3 --no-cpu-baseline --e2e-steps 2 ${BARGS} > gpurun_out/bench_${T}.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/bench_${T}.log').read().strip().splitlines()[-1]); print('ms/view', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()})" || tail -5 gpurun_out/bench_${T}.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_${T}.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
python - <<PY
import csv,collections
rows=list(csv.reader(open('gpurun_out/launches_${T}.csv')))
hdr=None;d=collections.OrderedDict()
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr and len(r)==len(hdr): d.setdefault(r[hdr.index('Kernel Name')].split('(')[0],[]).append(float(r[hdr.index('Metric Value')])/1e3)
for k,v in d.items(): print(f"{k:40s} n={len(v):3d} mean={sum(v)/len(v):8.1f} us")
PY
