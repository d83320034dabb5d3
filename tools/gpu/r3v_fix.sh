mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r3v_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3v_tests.log
for v in kernel inkernel kernel inkernel; do echo "FQB_OZ_FIXUP=$v"; FQB_OZ_FIXUP=$v timeout 600 python tools/step_jitter.py 3; done > gpurun_out/r3v_jit.txt 2>&1
FQB_PROFILE_RUNS=1 timeout 900 python tools/kernel_profile.py --config c4 --svd --runs 1 > gpurun_out/r3v_kprof.txt 2>&1
