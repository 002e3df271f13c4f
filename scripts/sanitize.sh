#!/bin/bash
# compute-sanitizer over every K6 variant, the sort and the backward replay
# (scripts/sanitize_driver.py).  Usage: scripts/sanitize.sh TAG
O=gpurun_out/${1:-r2s}/sanitizer
mkdir -p $O
for tool in memcheck racecheck synccheck initcheck; do
  timeout 600 compute-sanitizer --tool $tool --kernel-name regex=3stp --print-limit 50 \
     --log-file $O/$tool.txt python scripts/sanitize_driver.py > $O/$tool.stdout 2>&1
  echo "$tool rc=$?" >> $O/summary.txt
  tail -3 $O/$tool.txt >> $O/summary.txt
done
