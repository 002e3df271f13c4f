#!/bin/bash
mkdir -p gpurun_out
TAG=${TAG:-f2}
BENCH="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_preprocess|k_duplicate|k_onesweep|k_ranges|k_sort_hist" -s 12 -c 5 \
  -o gpurun_out/prof_front_${TAG} $BENCH > gpurun_out/ncu_front_${TAG}.log 2>&1
echo "front capture exit $?"
