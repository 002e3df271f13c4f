#!/bin/bash
O=gpurun_out/r2f; mkdir -p $O
./scripts/micro/cub_sort 6500000 45 > $O/cub_yardstick.txt 2>&1
timeout 1200 python scripts/sort_error_table.py $O/table1.json > $O/table1.log 2>&1; echo "table rc=$?" >> $O/table1.log
timeout 600 compute-sanitizer --tool initcheck --kernel-name regex=3stp --print-limit 20 --log-file $O/initcheck.txt python scripts/sanitize_driver.py hier > $O/initcheck.stdout 2>&1; echo "initcheck rc=$?" >> $O/initcheck.stdout
timeout 900 python bench.py --steps 40 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
