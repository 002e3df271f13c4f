#!/bin/bash
# row-culling A/B: parity subset, then C3/C4 with and without row culling
mkdir -p gpurun_out
T=${TAG:-ra}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider -k "exact64 or determin or c4_law or elongated" > gpurun_out/pytest_${T}.log 2>&1
echo "pytest exit $?"; tail -1 gpurun_out/pytest_${T}.log
for v in rows norows; do
  fl=""; [ $v = norows ] && fl="-DSTP_ROWS=0"
  STP_NVCC_EXTRA="$fl" python paper_2402_00525_b200/build.py --force > /dev/null 2>&1
  for c in C3 C3 C4; do
    timeout 600 python bench.py --config $c --steps 16 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_${T}.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/bench_${T}.log').read().strip().splitlines()[-1]); print('$v $c', 'ms/view', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()})"
  done
done
python paper_2402_00525_b200/build.py --force > /dev/null 2>&1
