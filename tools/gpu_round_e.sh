o=gpurun_out/r2e; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_adversarial.py tests/test_gpu_golden.py tests/test_gpu_guard.py -x -q > $o/gpu_tests.txt 2>&1; echo "gpu tests rc=$?"; tail -3 $o/gpu_tests.txt
HYB_FUSED_LEAN11=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_adversarial.py -x -q > $o/gpu_tests_lean11.txt 2>&1; echo "gpu tests lean11 rc=$?"; tail -2 $o/gpu_tests_lean11.txt
run() { # config mode
  case $2 in split) export HYB_AMF_SPLIT=1;; lean11) export HYB_FUSED_LEAN11=1;; esac
  timeout 300 python bench.py --config $1 --no-cpu-baseline > $o/bench_c$1_$2.json 2> $o/bench_c$1_$2.err
  unset HYB_AMF_SPLIT HYB_FUSED_LEAN11
  python - <<PY
import json
d=json.loads(open("$o/bench_c$1_$2.json").read().strip().splitlines()[-1])
print("C$1 $2", d["value"], d["ms_per_step"], d["roofline"]["kernel_ms"], d["clocks"]["sm_mhz"], d["clocks"]["samples"])
PY
}
for m in fused lean11 split fused lean11 split; do run 4 $m; done
for m in fused split fused split; do run 2 $m; run 3 $m; done
