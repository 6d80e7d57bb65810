# usage: tools/gpu_ab.sh <outdir> "<config:mode> ..."   mode in default|split|fused
o=$1; mkdir -p $o
for cm in $2; do
  c=${cm%%:*}; m=${cm##*:}
  case $m in split) export HYB_AMF_SPLIT=1;; fused) export HYB_AMF_FUSED=1;; esac
  timeout 300 python bench.py --config $c --no-cpu-baseline > $o/bench_c${c}_$m.json 2> $o/bench_c${c}_$m.err
  unset HYB_AMF_SPLIT HYB_AMF_FUSED
  python - <<PY
import json
try:
    d=json.loads(open("$o/bench_c${c}_$m.json").read().strip().splitlines()[-1])
    print("C$c $m", d["value"], d["ms_per_step"], d["roofline"]["kernel_ms"], d["clocks"]["sm_mhz"])
except Exception as e:
    print("C$c $m FAILED", e, open("$o/bench_c${c}_$m.err").read()[-500:])
PY
done
