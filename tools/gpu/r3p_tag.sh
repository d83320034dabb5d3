mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r3p_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3p_tests.log
timeout 600 python tools/step_jitter.py 6 > gpurun_out/r3p_jit.txt 2>&1
