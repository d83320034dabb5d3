set -x
mkdir -p gpurun_out
timeout 900 python tools/kernel_profile.py --config c4 --svd --runs 2 > gpurun_out/r28_kprof_c4.txt 2>&1
