set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r12_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/r12_gputest.log
timeout 900 python tools/step_jitter.py 5 > gpurun_out/r12_jitter.txt 2>&1
timeout 900 python tools/kernel_profile.py --config c4 --svd --runs 3 > gpurun_out/r12_kprof.txt 2>&1
