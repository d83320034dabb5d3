mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_chol.py -q -p no:cacheprovider -x > gpurun_out/r3e_chol.log 2>&1; echo "rc=$?" >> gpurun_out/r3e_chol.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bigcases.py tests/test_gpu_edge_parity.py -q -p no:cacheprovider -x > gpurun_out/r3e_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3e_tests.log
for v in reg blk reg blk; do echo "FQB_CHOL=$v"; FQB_CHOL=$v timeout 600 python tools/step_jitter.py 3; done > gpurun_out/r3e_jit.txt 2>&1
FQB_PROFILE_RUNS=1 timeout 900 python tools/kernel_profile.py --config c4 --svd --runs 1 > gpurun_out/r3e_kprof.txt 2>&1
