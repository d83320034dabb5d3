set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_bigcases.py -q -p no:cacheprovider > gpurun_out/r30_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r30_tests.log
timeout 600 python tools/step_jitter.py 8 > gpurun_out/r30_jit.txt 2>&1
FQB_OZ_QMN=0 timeout 600 python tools/step_jitter.py 8 > gpurun_out/r30_jit_qmn0.txt 2>&1
timeout 600 python tools/step_jitter.py 8 > gpurun_out/r30_jit_b.txt 2>&1
