#!/bin/bash
TAG=${1:-r2q}
bash scripts/r2_full.sh $TAG
timeout 1500 python scripts/sort_error_table.py gpurun_out/$TAG/table1.json > gpurun_out/$TAG/table1.log 2>&1; echo "table rc=$?" >> gpurun_out/$TAG/table1.log
