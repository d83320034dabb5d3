mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_int8_bgs.py -q -p no:cacheprovider --durations=4 > gpurun_out/r4c_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r4c_tests.log
