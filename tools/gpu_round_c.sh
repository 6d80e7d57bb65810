o=gpurun_out/r2c; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -x -q > $o/gpu_tests.txt 2>&1; echo "gpu tests rc=$?"; tail -15 $o/gpu_tests.txt
for c in 4 2 3 1; do
  for mode in fused split; do
    if [ $mode = split ]; then export HYB_AMF_SPLIT=1; else unset HYB_AMF_SPLIT; fi
    timeout 300 python bench.py --config $c --no-cpu-baseline > $o/bench_c${c}_$mode.json 2> $o/bench_c${c}_$mode.err
    python - <<PY
import json
d=json.loads(open("$o/bench_c${c}_$mode.json").read().strip().splitlines()[-1])
print("C$c $mode", d["value"], d["ms_per_step"], d["roofline"]["kernel_ms"], d["clocks"]["sm_mhz"], d["clocks"]["samples"])
PY
  done
done
unset HYB_AMF_SPLIT
