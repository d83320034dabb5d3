mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_int8_bgs.py tests/test_gpu_chol.py -q -p no:cacheprovider --durations=5 > gpurun_out/r3f_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3f_tests.log
