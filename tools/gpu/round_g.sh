set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cpp_dropin.py -q -p no:cacheprovider > gpurun_out/r7_dropin.log 2>&1; echo "rc=$?" >> gpurun_out/r7_dropin.log
timeout 900 python tools/step_jitter.py 12 > gpurun_out/r7_jitter.txt 2>&1
