#!/bin/bash
# ncu --set full (+ source) of the config-4 AMF kernels, and the growth-level trace.
o=gpurun_out/${1:-prof_grow}; mkdir -p $o
make trace > /dev/null 2>&1
timeout 300 python tools/trace_levels.py 4 > $o/trace_levels.txt 2>&1; cat $o/trace_levels.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:amf_ -c 2 -o $o/amf_c4 \
   python tools/hybrid_dev.py 4 1 > $o/ncu.log 2>&1; echo "ncu rc=$?"; tail -3 $o/ncu.log
