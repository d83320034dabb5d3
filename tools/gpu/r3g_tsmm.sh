mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tsmm.py -q -p no:cacheprovider -x > gpurun_out/r3g_tsmm.log 2>&1; echo "rc=$?" >> gpurun_out/r3g_tsmm.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bigcases.py tests/test_gpu_fp32.py tests/test_gpu_multirank.py tests/test_gpu_edge_parity.py tests/test_gpu_int8_bgs.py -q -p no:cacheprovider -x > gpurun_out/r3g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3g_tests.log
for v in 0 1 0 1; do echo "FQB_TSMM=$v"; FQB_TSMM=$v timeout 600 python tools/step_jitter.py 3; done > gpurun_out/r3g_jit.txt 2>&1
timeout 600 python tools/small_gemm_c4.py 1000 > gpurun_out/r3g_small.txt 2>&1
FQB_PROFILE_RUNS=1 timeout 900 python tools/kernel_profile.py --config c4 --svd --runs 1 > gpurun_out/r3g_kprof.txt 2>&1
