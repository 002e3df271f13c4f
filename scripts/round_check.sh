#!/bin/bash
# One GPU round trip: parity tests, smoke, default bench, ncu launch list and
# one full capture of the dominant kernel.  Outputs under gpurun_out/.
mkdir -p gpurun_out
TAG=${TAG:-r1}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt
timeout 900 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu_${TAG}.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_${TAG}.log
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench_${TAG}.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_${TAG}.log
if [ -z "$NO_NCU" ]; then
BENCH="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file gpurun_out/launches_${TAG}.csv $BENCH > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo "launch list exit $?" >> gpurun_out/ncu_launch_${TAG}.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_render -s 2 -c 1 \
  -o gpurun_out/prof_render_${TAG} $BENCH > gpurun_out/ncu_render_${TAG}.log 2>&1
echo "render capture exit $?" >> gpurun_out/ncu_render_${TAG}.log
fi
tail -3 gpurun_out/pytest_gpu_${TAG}.log; tail -2 gpurun_out/smoke_${TAG}.log; tail -2 gpurun_out/bench_${TAG}.log
