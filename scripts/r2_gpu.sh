#!/bin/bash
# Round-2 GPU pass: smoke, GPU tests, bench, launch list.  Usage: scripts/r2_gpu.sh TAG [pytest-args]
TAG=${1:-r2a}; shift
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
nproc > $O/nproc.txt; free -g >> $O/nproc.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=25 "$@" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 40 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 120 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --streams 1 --no-cpu-baseline --e2e-steps 1 > $O/ncu_bench.log 2>&1
echo done
