o=gpurun_out/r2d; mkdir -p $o
timeout 900 ncu --set full --import-source on --clock-control none -k regex:amf_fused -c 1 -o $o/fused_c4 python tools/hybrid_dev.py 4 1 > $o/ncu_c4.log 2>&1; echo "ncu rc=$?"; tail -3 $o/ncu_c4.log
