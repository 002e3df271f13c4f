#!/bin/bash
# A/B of compile-time knobs on the GPU: scripts/ab.sh TAG "variant1:-DX=1 -DY=2" "variant2:..."
# (variants are built HERE first with build.py --variant; this runs on the box)
TAG=$1; shift
O=gpurun_out/$TAG; mkdir -p $O
run() {  # name lib
  for rep in ${AB_REPS:-1 2}; do
    STP_LIB_VARIANT=$2 timeout 300 python bench.py --steps 64 --warmup 5 --no-cpu-baseline --e2e-steps 2 > $O/bench_$1_$rep.json 2>$O/bench_$1_$rep.err
    python -c "import json,sys; d=json.loads(open('$O/bench_$1_$rep.json').read().strip().splitlines()[-1]); print('$1', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['kernel_ms'].items()})" >> $O/summary.txt 2>&1
  done
}
run base ""
for v in "$@"; do run $v paper_2402_00525_b200/variants/libstp_$v.so; done
cat $O/summary.txt
