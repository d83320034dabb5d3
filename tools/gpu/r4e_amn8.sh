mkdir -p gpurun_out
for l in 500 1000 1900; do timeout 300 python tools/amn_once.py $l 5; done > gpurun_out/r4e_amn.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r4e_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r4e_tests.log
timeout 600 python tools/step_jitter.py 5 > gpurun_out/r4e_jit.txt 2>&1
FQB_PROFILE_RUNS=1 timeout 900 python tools/kernel_profile.py --config c4 --svd --runs 1 > gpurun_out/r4e_kprof.txt 2>&1
