#!/bin/bash
# Build locally first (fail fast), then run a GPU script: scripts/gpu.sh TAG script.sh [timeout]
set -e
cd /root/repo
python paper_2402_00525_b200/build.py --force > /tmp/build.log 2>&1 || { grep -E "error" /tmp/build.log | head; exit 1; }
T=$1; S=$2; TO=${3:-1500}
timeout $((TO + 900)) /usr/local/graft/bin/gpurun --timeout $TO -- "TAG=$T bash $S" 2>&1 | tail -${TAIL:-16}
