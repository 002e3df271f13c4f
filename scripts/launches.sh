#!/bin/bash
# ncu launch list (per-kernel durations) of a short bench run: CFG (default C3)
mkdir -p gpurun_out
T=${TAG:-ll}
for c in ${CFGS:-C3}; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c ${NK:-60} --csv --log-file gpurun_out/launches_${T}_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
python - <<PY
import csv,collections
rows=list(csv.reader(open('gpurun_out/launches_${T}_$c.csv')))
hdr=None;d=collections.OrderedDict()
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr and len(r)==len(hdr): d.setdefault(r[hdr.index('Kernel Name')].split('(')[0],[]).append(float(r[hdr.index('Metric Value')])/1e3)
for k,v in d.items(): print("$c", f"{k:40s} n={len(v):3d} mean={sum(v)/len(v):8.1f} us")
PY
done
