#!/bin/bash
# C4 sort A/B of compile-time variants: VARIANTS="name:flags;..."
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "${VARIANTS}"
for v in "${VS[@]}"; do
  n=${v%%:*}; fl=${v#*:}
  STP_NVCC_EXTRA="$fl" python paper_2402_00525_b200/build.py --force > /dev/null 2>&1 || { echo "$n build failed"; continue; }
  timeout 600 python bench.py --config C4 --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_c4_${n}.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bench_c4_${n}.log').read().strip().splitlines()[-1]); print('$n', 'ms/view', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()})"
done
python paper_2402_00525_b200/build.py --force > /dev/null 2>&1
