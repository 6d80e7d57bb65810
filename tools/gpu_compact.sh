#!/bin/bash
# Compact growth windows: GPU tests of the path, config-3 A/B, ncu of the AMF kernels.
o=gpurun_out/${1:-compact}; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_compact.py tests/test_gpu_paths.py -q -x > $o/tests.txt 2>&1; echo "tests rc=$?"; tail -3 $o/tests.txt
HYB_LIB=libhybrid_cuda_alt.so timeout 900 python -m pytest tests/test_gpu_compact.py -q -x > $o/tests_alt.txt 2>&1; echo "alt tests rc=$?"; tail -1 $o/tests_alt.txt
for i in 1 2; do
  echo -n "T=0 "; HYB_COMPACT_T=0 tools/bench_all.sh 3
  echo -n "coop "; tools/bench_all.sh 3
  echo -n "lane "; HYB_LIB=libhybrid_cuda_alt.so tools/bench_all.sh 3
done 2>&1 | tee $o/ab.txt
for v in coop lane; do
  if [ $v = lane ]; then export HYB_LIB=libhybrid_cuda_alt.so; fi
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:amf --csv python tools/batch_dev.py 512 1 > $o/ncu_$v.csv 2>&1
done
unset HYB_LIB
timeout 600 ncu --set full --import-source on --clock-control none -k regex:amf -o $o/full_amf python tools/batch_dev.py 512 1 > $o/ncu.log 2>&1; echo "ncu rc=$?"
