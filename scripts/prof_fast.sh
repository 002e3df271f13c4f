#!/bin/bash
mkdir -p gpurun_out
T=${TAG:-pf}
BENCH="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KERN:-k_render_fast} -s 2 -c 1 \
  -o gpurun_out/prof_${T} $BENCH > gpurun_out/ncu_${T}.log 2>&1
echo "capture exit $?"
