#!/bin/bash
bash scripts/quick2.sh
T=${TAG:-k13}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_preprocess|k_duplicate" -s 4 -c 2 \
  -o gpurun_out/prof_${T} python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_${T}.log 2>&1
echo "capture exit $?"
