#!/bin/bash
# K6 per-phase warp-cycle split (instrumented build, never a bench number),
# then the work counters from a separate build.
mkdir -p gpurun_out
STP_NVCC_EXTRA=-DSTP_PHASE_PROF python paper_2402_00525_b200/build.py --force > /dev/null 2>&1
timeout 300 python scripts/phase_prof.py ${CFG:-C3} > gpurun_out/phase_${TAG:-x}.log 2>&1
STP_NVCC_EXTRA=-DSTP_WORK_STATS python paper_2402_00525_b200/build.py --force > /dev/null 2>&1
timeout 300 python scripts/phase_prof.py ${CFG:-C3} >> gpurun_out/phase_${TAG:-x}.log 2>&1
cat gpurun_out/phase_${TAG:-x}.log
python paper_2402_00525_b200/build.py --force > /dev/null 2>&1
