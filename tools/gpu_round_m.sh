o=gpurun_out/r2m; mkdir -p $o
for lib in libhybrid_cuda_alt1.so libhybrid_cuda_alt2.so; do
HYB_LIB=$lib timeout 600 python -m pytest tests/test_gpu_paths.py -x -q -k SPLIT > $o/t_$lib.txt 2>&1; echo "$lib tests rc=$?"; tail -1 $o/t_$lib.txt; done
for lib in libhybrid_cuda.so libhybrid_cuda_alt1.so libhybrid_cuda_alt2.so libhybrid_cuda.so libhybrid_cuda_alt1.so libhybrid_cuda_alt2.so; do
HYB_LIB=$lib timeout 300 python bench.py --config 4 --no-cpu-baseline > $o/bench_c4.json 2> $o/bench_c4.err
python - <<PY
import json
d=json.loads(open("$o/bench_c4.json").read().strip().splitlines()[-1])
print("C4 $lib", d["value"], d["ms_per_step"], d["roofline"]["kernel_ms"])
PY
done
