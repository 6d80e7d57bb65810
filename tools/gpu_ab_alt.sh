#!/bin/bash
# A/B of alternative builds (make alt ALTDEF=...; libhybrid_cuda_alt<N>.so) against the shipped library.
# usage: tools/gpu_ab_alt.sh "<alt numbers>" [configs]
for i in 1 2; do
  echo -n "base  "; tools/bench_all.sh ${2:-4}
  for v in $1; do echo -n "alt$v  "; HYB_LIB=libhybrid_cuda_alt$v.so tools/bench_all.sh ${2:-4}; done
done 2>&1 | tee gpurun_out/ab_alt.txt
