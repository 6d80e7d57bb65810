o=gpurun_out/r2j; mkdir -p $o
for lib in libhybrid_cuda.so libhybrid_cuda_alt1.so libhybrid_cuda_alt2.so libhybrid_cuda.so libhybrid_cuda_alt1.so; do
HYB_LIB=$lib timeout 300 python bench.py --config 4 --no-cpu-baseline > $o/bench_c4.json 2> $o/bench_c4.err
python - <<PY
import json
d=json.loads(open("$o/bench_c4.json").read().strip().splitlines()[-1])
print("C4 $lib", d["value"], d["ms_per_step"], d["roofline"]["kernel_ms"], d["clocks"]["sm_mhz"])
PY
done
