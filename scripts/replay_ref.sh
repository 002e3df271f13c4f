#!/bin/bash
# Run the reference's own test files through the B200 render path
# (splatsort_plugin), one junit report per file.  Usage: scripts/replay_ref.sh OUTDIR [files]
O=${1:-gpurun_out/replay}; shift
mkdir -p $O
ROOT=$(pwd)
FILES=${@:-test_rasterizer.py test_acceptance.py test_gradients.py test_metrics.py}
for f in $FILES; do
  (cd baseline/_ref && PYTHONPATH=$ROOT/baseline/_ref:$ROOT timeout 1800 python -m pytest \
     -p paper_2402_00525_b200.splatsort_plugin -p no:cacheprovider -q -rA \
     --junitxml=$ROOT/$O/${f%.py}.xml tests/$f) > $O/${f%.py}.log 2>&1
  echo "$f rc=$?" >> $O/summary.txt
done
