#!/bin/bash
O=gpurun_out/r2g; mkdir -p $O
bash scripts/ab.sh r2g_ab k6w2r112 k6w1r112 k6w2r104 k6minb5
timeout 1200 python scripts/sort_error_table.py $O/table1.json > $O/table1.log 2>&1; echo "table rc=$?" >> $O/table1.log
timeout 1200 python scripts/reference_cpu_point.py $O/reference_python_C3.json C3 5 48 > $O/refpt.log 2>&1; echo "refpt rc=$?" >> $O/refpt.log
