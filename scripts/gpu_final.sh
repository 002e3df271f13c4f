#!/bin/bash
# Round-end evidence on one box: smoke, every GPU test, the default bench,
# per-kernel ncu of a C3 view, Table 1, C2 / C5 / C4 benches, sanitizer.
# Usage: scripts/gpu_final.sh TAG
TAG=${1:-final}
O=gpurun_out/$TAG; mkdir -p $O
NO_NCU= bash scripts/gpu_full.sh $TAG
timeout 900 python scripts/sort_error_table.py $O/table1.json > $O/table1.log 2>&1
for c in C2 C5 C4; do
  timeout 600 python bench.py --config $c --steps 16 --warmup 4 --no-cpu-baseline --e2e-steps 4 > $O/bench_$c.json 2> $O/bench_$c.err
done
O2=gpurun_out/$TAG/sanitizer; mkdir -p $O2
for tool in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $tool --kernel-name regex=3stp --print-limit 50 \
     --log-file $O2/$tool.txt python scripts/sanitize_driver.py > $O2/$tool.stdout 2>&1
  echo "$tool rc=$?" >> $O2/summary.txt
  tail -3 $O2/$tool.txt >> $O2/summary.txt
done
echo done
