#!/bin/bash
# ncu evidence for one bench view: launch list + full captures. Outputs in gpurun_out/.
mkdir -p gpurun_out
TAG=${TAG:-r1}
BENCH="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv \
  --log-file gpurun_out/launches_${TAG}.csv $BENCH > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo "launch list exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_render -s 1 -c 1 \
  -o gpurun_out/prof_render_${TAG} $BENCH > gpurun_out/ncu_render_${TAG}.log 2>&1
echo "render capture exit $?"
timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"k_preprocess|k_duplicate|k_onesweep|k_ranges" -s 10 -c 4 \
  -o gpurun_out/prof_front_${TAG} $BENCH > gpurun_out/ncu_front_${TAG}.log 2>&1
echo "front capture exit $?"
ls -la gpurun_out/
