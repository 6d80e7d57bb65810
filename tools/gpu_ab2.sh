#!/bin/bash
# usage: tools/gpu_ab2.sh <tag> <alt.so> "<configs>" [extra env for a third arm, e.g. HYB_AMF_FUSED=1]
# parity tests of the default build, then alternating bench of the default and the alt build.
o=gpurun_out/$1; alt=$2; cfgs=${3:-"1 2 3 4"}; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py tests/test_gpu_adversarial.py -x -q > $o/tests.txt 2>&1; echo "tests rc=$?"; tail -2 $o/tests.txt
for rep in 1 2; do
  for c in $cfgs; do
    echo -n "base "; tools/bench_all.sh $c
    echo -n "alt  "; HYB_LIB=$alt tools/bench_all.sh $c
    if [ -n "$4" ]; then echo -n "env  "; env $4 tools/bench_all.sh $c; fi
  done
done
