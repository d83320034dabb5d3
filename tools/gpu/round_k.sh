set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r11_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/r11_gputest.log
FQB_OZ_Q=0 timeout 900 python tools/step_jitter.py 4 > gpurun_out/r11_jitter_q0.txt 2>&1
timeout 900 python tools/step_jitter.py 6 > gpurun_out/r11_jitter_q1.txt 2>&1
timeout 900 python tools/kernel_profile.py --config c4 --svd --runs 3 > gpurun_out/r11_kprof.txt 2>&1
