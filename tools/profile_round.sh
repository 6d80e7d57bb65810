#!/bin/bash
# Evidence for profiles/r1 (run on the GPU box): GPU tests, the default bench line, the reference arm,
# the ncu launch list of the bench command, and ncu --set full captures of configs 1 / 2 / 4.
# usage: tools/profile_round.sh <tag>   (outputs under gpurun_out/prof_<tag>/)
tag=${1:-v}
o=gpurun_out/prof_$tag
mkdir -p $o
timeout 600 python -m pytest tests -m gpu -q > $o/gpu_tests.txt 2>&1; echo "gpu tests rc=$?"; tail -1 $o/gpu_tests.txt
timeout 900 python bench.py > $o/bench_config1.json 2> $o/bench.err; echo "bench rc=$?"; tail -c 400 $o/bench_config1.json
timeout 900 python bench.py --impl reference > $o/bench_reference.json 2> $o/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches_config1.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $o/ncu_launch.log 2>&1; echo "launch list rc=$?"
for c in 1 2 4; do
  timeout 900 ncu --set full --import-source on --clock-control none -o $o/full_config$c \
      python tools/hybrid_dev.py $c 1 > $o/ncu_full_$c.log 2>&1; echo "ncu full config $c rc=$?"
done
