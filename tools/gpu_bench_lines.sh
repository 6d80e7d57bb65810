#!/bin/bash
# Bench lines of every configuration (the default line with its CPU baseline, the others without).
# usage: tools/gpu_bench_lines.sh <tag>
o=gpurun_out/bench_${1:-x}; mkdir -p $o
timeout 900 python bench.py > $o/bench_config4.json 2> $o/bench.err; echo "bench rc=$?"; tail -c 400 $o/bench_config4.json
for c in 0 1 2 3; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $o/bench_config$c.json 2>> $o/bench.err; echo "bench config $c rc=$?"
done
