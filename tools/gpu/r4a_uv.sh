mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fixed_rank_device.py tests/test_gpu_bigcases.py tests/test_gpu_fullsize.py tests/test_cpp_dropin.py tests/test_gpu_experiment.py tests/test_gpu_eig.py -q -p no:cacheprovider -x > gpurun_out/r4a_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r4a_tests.log
FQB_HOST_STATS=1 timeout 900 python tools/e2e_probe.py 3 > gpurun_out/r4a_e2e.txt 2>&1
