o=gpurun_out/r2i; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py tests/test_gpu_adversarial.py -x -q > $o/gpu_tests.txt 2>&1; echo "gpu tests rc=$?"; tail -2 $o/gpu_tests.txt
bash tools/gpu_ab.sh $o "4:fused 4:split 3:fused 3:split 2:fused 2:split 4:fused 4:split 3:fused 3:split"
