mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_chol.py tests/test_gpu_parity.py tests/test_gpu_edge_parity.py tests/test_gpu_bigcases.py tests/test_gpu_fp32.py tests/test_gpu_fixed_rank_device.py -q -p no:cacheprovider -x > gpurun_out/r3u_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3u_tests.log
timeout 600 python tools/step_jitter.py 6 > gpurun_out/r3u_jit.txt 2>&1
FQB_PROFILE_RUNS=1 timeout 900 python tools/kernel_profile.py --config c4 --svd --runs 1 > gpurun_out/r3u_kprof.txt 2>&1
