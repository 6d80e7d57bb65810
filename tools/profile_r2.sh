#!/bin/bash
# Round-2 evidence (run on the GPU box): GPU tests, the default bench line (config 4), the reference arm,
# per-config bench lines, the ncu launch list of the bench command, and ncu --set full captures of
# configs 1-4.  usage: tools/profile_r2.sh <tag>   (outputs under gpurun_out/prof_<tag>/)
tag=${1:-v}
o=gpurun_out/prof_$tag
mkdir -p $o
nvidia-smi > $o/nvidia_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > $o/gpu_tests.txt 2>&1; echo "gpu tests rc=$?"; tail -1 $o/gpu_tests.txt
timeout 900 python bench.py > $o/bench_config4.json 2> $o/bench.err; echo "bench rc=$?"; tail -c 300 $o/bench_config4.json
timeout 900 python bench.py --impl reference > $o/bench_reference.json 2> $o/bench_ref.err; echo "ref rc=$?"; tail -c 300 $o/bench_reference.json
for c in 0 1 2 3; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $o/bench_config$c.json 2>> $o/bench.err; echo "bench config $c rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $o/launches_config4.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $o/ncu_launch.log 2>&1; echo "launch list rc=$?"
for c in 1 2 3 4; do
  if [ $c = 3 ]; then cmd="python tools/batch_dev.py 512 1"; else cmd="python tools/hybrid_dev.py $c 1"; fi  # config 3 = the 512-slice stack
  timeout 900 ncu --set full --import-source on --clock-control none -o $o/full_config$c \
      $cmd > $o/ncu_full_$c.log 2>&1; echo "ncu full config $c rc=$?"
  # summaries are made here (gpurun merges at most 64 MiB back): only config 4's report travels
  (echo "# ncu --set full --clock-control none, $cmd, tag $tag"; python tools/ncu_report.py $o/full_config$c.ncu-rep) > $o/ncu_full_config$c.txt 2>&1
  python tools/ncu_counters.py $c $o/full_config$c.ncu-rep > /dev/null 2>&1
  if [ $c != 4 ]; then rm -f $o/full_config$c.ncu-rep; fi
done
cp profiles/ncu_counters.json $o/ncu_counters.json
timeout 600 python tools/strip_projection.py 2 4 > $o/strip_projection.txt 2>&1; cat $o/strip_projection.txt
timeout 300 python tools/strip_stages.py 4 > $o/strip_stages.txt 2>&1; tail -12 $o/strip_stages.txt
