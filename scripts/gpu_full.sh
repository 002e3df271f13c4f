#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_full_${TAG:-x}.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_full_${TAG:-x}.log; tail -4 gpurun_out/pytest_full_${TAG:-x}.log
