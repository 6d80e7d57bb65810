o=gpurun_out/r2l; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_context.py tests/test_gpu_multi.py tests/test_capi.py -x -q > $o/gpu_tests.txt 2>&1; echo "gpu tests rc=$?"; tail -3 $o/gpu_tests.txt
for c in 4 1 2; do
timeout 300 python bench.py --config $c --no-cpu-baseline > $o/bench_c$c.json 2> $o/bench_c$c.err
python - <<PY
import json
d=json.loads(open("$o/bench_c$c.json").read().strip().splitlines()[-1])
print("C$c", d["value"], d["ms_per_step"], "e2e", d["e2e"]["value"], d["e2e"]["ms_per_step"], "sync", d["e2e"].get("synchronous"))
PY
done
