set -x
o=gpurun_out/r2a; mkdir -p $o
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $o/smi.txt
tools/int_peak > $o/int_peak.json 2>&1; echo "int_peak rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > $o/gpu_tests.txt 2>&1; echo "gpu tests rc=$?"; tail -3 $o/gpu_tests.txt
timeout 600 python bench.py > $o/bench.json 2> $o/bench.err; echo "bench rc=$?"; tail -c 3000 $o/bench.json
timeout 600 python bench.py --impl reference > $o/ref.json 2> $o/ref.err; echo "ref rc=$?"; tail -c 1500 $o/ref.json
