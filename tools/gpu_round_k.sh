o=gpurun_out/r2k; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py tests/test_gpu_adversarial.py tests/test_gpu_golden.py tests/test_gpu_guard.py tests/test_gpu_partition.py -x -q > $o/gpu_tests.txt 2>&1; echo "gpu tests rc=$?"; tail -2 $o/gpu_tests.txt
bash tools/gpu_ab.sh $o "4:default 3:default 2:split 4:default 3:default"
