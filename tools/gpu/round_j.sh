set -x
mkdir -p gpurun_out
FQB_ALLOC_STATS=1 FQB_HOST_STATS=1 timeout 900 python tools/step_jitter.py 8 > gpurun_out/r10_alloc.txt 2>&1
timeout 900 python tools/kernel_profile.py --config c4 --svd --runs 4 > gpurun_out/r10_kprof.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r10_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/r10_gputest.log
