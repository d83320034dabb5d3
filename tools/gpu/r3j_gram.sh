mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tsmm.py tests/test_gpu_parity.py tests/test_gpu_bigcases.py tests/test_gpu_fp32.py -q -p no:cacheprovider -x > gpurun_out/r3j_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3j_tests.log
for v in 0 1 0 1; do echo "FQB_TSMM=$v"; FQB_TSMM=$v timeout 600 python tools/step_jitter.py 3; done > gpurun_out/r3j_jit.txt 2>&1
