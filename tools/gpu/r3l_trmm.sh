mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tsmm.py tests/test_gpu_parity.py tests/test_gpu_bigcases.py -q -p no:cacheprovider -x > gpurun_out/r3l_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3l_tests.log
timeout 600 python tools/small_gemm_c4.py 1000 > gpurun_out/r3l_small.txt 2>&1
for v in 0 1 0 1; do echo "FQB_TSMM=$v"; FQB_TSMM=$v timeout 600 python tools/step_jitter.py 3; done > gpurun_out/r3l_jit.txt 2>&1
timeout 300 python tools/tsmm_once.py > gpurun_out/r3l_once.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:k_ts_ -c 8 -o gpurun_out/r3l_ncu_tsmm python tools/tsmm_once.py > gpurun_out/r3l_ncu.log 2>&1
