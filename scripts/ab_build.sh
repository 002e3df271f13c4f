#!/bin/bash
# A/B of compile-time variants on one box: VARIANTS="name:flags;name2:flags2"
# each variant: rebuild with STP_NVCC_EXTRA, exact parity subset, C3 bench.
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "${VARIANTS}"
for v in "${VS[@]}"; do
  n=${v%%:*}; fl=${v#*:}
  STP_NVCC_EXTRA="$fl" python paper_2402_00525_b200/build.py --force > gpurun_out/build_${n}.log 2>&1 || { echo "$n build failed"; continue; }
  if [ -z "$NOTEST" ]; then
    timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -p no:cacheprovider -k "exact64 or determin" > gpurun_out/pytest_${n}.log 2>&1
    echo "$n pytest exit $?"; tail -1 gpurun_out/pytest_${n}.log
  fi
  for rep in 1 2; do
    timeout 300 python bench.py --steps 32 --warmup 3 --no-cpu-baseline --e2e-steps 2 ${BARGS} > gpurun_out/bench_${n}.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/bench_${n}.log').read().strip().splitlines()[-1]); print('$n', 'ms/view', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()})" || tail -5 gpurun_out/bench_${n}.log
  done
done
python paper_2402_00525_b200/build.py --force > /dev/null 2>&1
