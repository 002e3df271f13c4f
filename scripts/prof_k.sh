#!/bin/bash
# one ncu --set full capture per kernel in KERNS (regex list), C3 bench
mkdir -p gpurun_out
T=${TAG:-pk}
BENCH="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 ${BARGS}"
for k in ${KERNS:-k_preprocess}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s ${SKIP:-2} -c 1 \
    -o gpurun_out/prof_${T}_$k $BENCH > gpurun_out/ncu_${T}_$k.log 2>&1
  echo "$k capture exit $?"
done
