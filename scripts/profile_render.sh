#!/bin/bash
mkdir -p gpurun_out
TAG=${TAG:-r1b}
BENCH="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_render -s 1 -c 1 \
  -o gpurun_out/prof_render_${TAG} $BENCH > gpurun_out/ncu_render_${TAG}.log 2>&1
echo "render capture exit $?"
