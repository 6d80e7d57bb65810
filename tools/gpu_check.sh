#!/bin/bash
# One GPU pass over the current tree: GPU tests, the default bench line, and the per-config summary.
# usage: tools/gpu_check.sh <tag>   (outputs under gpurun_out/<tag>/)
tag=${1:-chk}
o=gpurun_out/$tag; mkdir -p $o
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $o/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $o/gpu_tests.txt 2>&1; echo "gpu tests rc=$?"; tail -3 $o/gpu_tests.txt
timeout 600 python bench.py > $o/bench.json 2> $o/bench.err; echo "bench rc=$?"; tail -c 600 $o/bench.json
timeout 900 tools/bench_all.sh > $o/bench_all.txt 2>&1; cat $o/bench_all.txt
