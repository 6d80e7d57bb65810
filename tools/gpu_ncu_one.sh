#!/bin/bash
# usage: tools/gpu_ncu_one.sh <tag> <kernel regex> <config> [lib]  -- ncu --set full (+source) of one kernel
o=gpurun_out/$1; mkdir -p $o
HYB_LIB=${4:-libhybrid_cuda.so} timeout 900 ncu --set full --import-source on --clock-control none -k regex:$2 -c ${5:-1} -o $o/prof \
   python tools/hybrid_dev.py $3 1 > $o/ncu.log 2>&1; echo "ncu rc=$?"; tail -2 $o/ncu.log
