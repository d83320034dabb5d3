set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cpp_dropin.py tests/test_gpu_rawio.py -q -p no:cacheprovider > gpurun_out/r8_dropin.log 2>&1; echo "rc=$?" >> gpurun_out/r8_dropin.log
FQB_HOST_STATS=1 timeout 900 python tools/step_jitter.py 8 > gpurun_out/r8_jitter.txt 2>&1
timeout 900 python tools/kernel_profile.py --config c4 --svd --runs 6 > gpurun_out/r8_kprof.txt 2>&1
