#!/bin/bash
# Per-kernel ncu evidence for one C3 view: a --set full capture of every
# in-repo kernel of the second view bench.py renders (K0..K6, 16 launches),
# plus the launch list of the same command.  Usage: scripts/ncu_capture.sh TAG [bench args]
TAG=${1:-r2c}; shift
O=gpurun_out/$TAG
mkdir -p $O
BENCH="python bench.py --steps 2 --warmup 3 --streams 1 --no-cpu-baseline --e2e-steps 1 $@"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_" \
  --launch-skip 16 --launch-count 16 -o $O/full $BENCH > $O/ncu_full.log 2>&1
echo "full capture rc=$?" >> $O/ncu_full.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file $O/launches.csv $BENCH > $O/ncu_launches.log 2>&1
echo "launches rc=$?" >> $O/ncu_launches.log
