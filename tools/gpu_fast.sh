#!/bin/bash
# Fast growth levels (zero / 255 bit planes): GPU tests, config-4 A/B against the plain levels.
# usage: tools/gpu_fast.sh <tag> [quick]
o=gpurun_out/${1:-fast}; mkdir -p $o
if [ "$2" = quick ]; then
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_adversarial.py tests/test_gpu_paths.py -m gpu -q -x > $o/tests.txt 2>&1; echo "tests rc=$?"; tail -3 $o/tests.txt
else
  timeout 1200 python -m pytest tests -m gpu -q -x > $o/tests.txt 2>&1; echo "tests rc=$?"; tail -3 $o/tests.txt
fi
for i in 1 2; do
  echo -n "plain "; HYB_GROW_FAST=0 tools/bench_all.sh 4
  echo -n "fast  "; tools/bench_all.sh 4
done 2>&1 | tee $o/ab.txt
