#!/bin/bash
# usage: tools/gpu_ab3.sh <tag> "<lib:ENV=V,...> ..." "<configs>"  -- parity of each variant's forced paths,
# then alternating benches: the default build first, then each variant (lib + env), twice.
o=gpurun_out/$1; mkdir -p $o; vars=$2; cfgs=${3:-"2 3 4"}
for v in $vars; do
  lib=${v%%:*}
  HYB_LIB=$lib timeout 900 python -m pytest tests/test_gpu_paths.py -x -q > $o/t_$lib.txt 2>&1; echo "$lib paths rc=$?"; tail -1 $o/t_$lib.txt
done
for rep in 1 2; do
  for c in $cfgs; do
    echo -n "base          "; tools/bench_all.sh $c
    for v in $vars; do
      lib=${v%%:*}; ev=${v#*:}; [ "$ev" = "$v" ] && ev=""
      echo -n "$v "; env HYB_LIB=$lib ${ev//,/ } tools/bench_all.sh $c
    done
  done
done
