#!/bin/bash
# C4 (6M at 4K) bench per knob variant: scripts/ab_c4.sh TAG v1 v2 ...
TAG=$1; shift
O=gpurun_out/$TAG; mkdir -p $O
for v in base "$@"; do
  lib=""; [ "$v" = base ] || lib=paper_2402_00525_b200/variants/libstp_$v.so
  STP_LIB_VARIANT=$lib timeout 300 python bench.py --config C4 --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $O/c4_$v.json 2> $O/c4_$v.err
  python -c "import json; d=json.loads(open('$O/c4_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],3), {k: round(x,3) for k,x in d['kernel_ms'].items()})" >> $O/summary.txt 2>&1
done
cat $O/summary.txt
