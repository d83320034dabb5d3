mkdir -p gpurun_out
timeout 600 python tools/small_gemm_c4.py 1000 > gpurun_out/r3h_small.txt 2>&1
timeout 300 python tools/tsmm_once.py > gpurun_out/r3h_once.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:k_ts_ -c 8 -o gpurun_out/r3h_ncu_tsmm python tools/tsmm_once.py > gpurun_out/r3h_ncu.log 2>&1
