o=gpurun_out/r2g; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py -x -q > $o/gpu_tests.txt 2>&1; echo "gpu tests rc=$?"; tail -2 $o/gpu_tests.txt
for i in 1 2; do
timeout 300 python bench.py --config 4 --no-cpu-baseline > $o/bench_c4.json 2> $o/bench_c4.err
python - <<PY
import json
d=json.loads(open("$o/bench_c4.json").read().strip().splitlines()[-1])
print("C4", d["value"], d["ms_per_step"], d["roofline"]["kernel_ms"], d["clocks"]["sm_mhz"], d["clocks"]["samples"])
PY
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:amf_grow -c 1 -o $o/grow_c4 python tools/hybrid_dev.py 4 1 > $o/ncu_c4.log 2>&1; echo "ncu rc=$?"
