mkdir -p gpurun_out
timeout 600 python tools/ozaki_ab.py "FQB_OZ_PAIR=1" "FQB_OZ_PAIR=1" > gpurun_out/r4f_ab.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r4f_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r4f_tests.log
timeout 600 python tools/step_jitter.py 5 > gpurun_out/r4f_jit.txt 2>&1
FQB_PROFILE_RUNS=1 timeout 900 python tools/kernel_profile.py --config c4 --svd --runs 1 > gpurun_out/r4f_kprof.txt 2>&1
