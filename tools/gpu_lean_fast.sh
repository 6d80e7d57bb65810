#!/bin/bash
# Bit-plane levels on the lean growth variant (HYB_GROW_FAST_LEAN=1): path tests and config 2 / 3 A/B.
o=gpurun_out/lean_fast; mkdir -p $o
HYB_GROW_FAST_LEAN=1 timeout 900 python -m pytest "tests/test_gpu_paths.py::test_amf_paths_vs_oracle[HYB_AMF_SPLIT]" tests/test_gpu_compact.py -m gpu -q -x > $o/tests.txt 2>&1; echo "tests rc=$?"; tail -3 $o/tests.txt
for i in 1 2; do
  echo -n "default         "; tools/bench_all.sh 2
  echo -n "split           "; HYB_AMF_SPLIT=1 tools/bench_all.sh 2
  echo -n "split lean-fast "; HYB_AMF_SPLIT=1 HYB_GROW_FAST_LEAN=1 tools/bench_all.sh 2
  echo -n "default         "; tools/bench_all.sh 3
  echo -n "lean-fast       "; HYB_GROW_FAST_LEAN=1 tools/bench_all.sh 3
done 2>&1 | tee $o/ab.txt
