#!/bin/bash
# work counters only (instrumented build), per config
mkdir -p gpurun_out
STP_NVCC_EXTRA=-DSTP_WORK_STATS python paper_2402_00525_b200/build.py --force > /dev/null 2>&1
for c in ${CFGS:-C3}; do timeout 300 python scripts/phase_prof.py $c 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$c', json.dumps(d['stats']))"; done > gpurun_out/stats_${TAG:-x}.log
cat gpurun_out/stats_${TAG:-x}.log
python paper_2402_00525_b200/build.py --force > /dev/null 2>&1
