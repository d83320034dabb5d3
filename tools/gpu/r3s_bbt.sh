mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_bigcases.py tests/test_gpu_fullsize.py tests/test_gpu_eig.py tests/test_gpu_int8_bgs.py tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/r3s_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3s_tests.log
timeout 600 python tools/step_jitter.py 6 > gpurun_out/r3s_jit.txt 2>&1
