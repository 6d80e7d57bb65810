set -x
o=gpurun_out/r2b; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_cpp_host.py tests/test_gpu_context.py tests/test_gpu_parity.py -x -q > $o/gpu_tests.txt 2>&1; echo "gpu tests rc=$?"; tail -15 $o/gpu_tests.txt
timeout 600 python bench.py --no-cpu-baseline > $o/bench.json 2> $o/bench.err; echo "bench rc=$?"; tail -c 1500 $o/bench.json
