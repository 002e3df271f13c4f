#!/bin/bash
# smoke, GPU tests (incl. the reference replay), bench, per-kernel ncu.  Usage: scripts/gpu_full.sh TAG
TAG=${1:-r2c}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -rs -rf --durations=30 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 40 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
[ -n "$NO_NCU" ] || bash scripts/ncu_capture.sh $TAG
echo done
