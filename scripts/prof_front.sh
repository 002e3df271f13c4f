#!/bin/bash
mkdir -p gpurun_out
T=${TAG:-fr}
./scripts/micro/cub_sort 6500000 45 > gpurun_out/cub_${T}.log 2>&1
./scripts/micro/cub_sort 6500000 40 >> gpurun_out/cub_${T}.log 2>&1
./scripts/micro/cub_sort 6500000 32 >> gpurun_out/cub_${T}.log 2>&1
cat gpurun_out/cub_${T}.log
BENCH="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_preprocess|k_duplicate|k_onesweep|k_ranges|k_sort_hist" -s 30 -c 5 \
  -o gpurun_out/prof_${T} $BENCH > gpurun_out/ncu_${T}.log 2>&1
echo "capture exit $?"
