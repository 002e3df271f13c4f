#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider -k "${K}" 2>&1 | tail -3
