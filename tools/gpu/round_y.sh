set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ozaki.py -q -p no:cacheprovider -k "mn or again or sliced" > gpurun_out/r26_mn.log 2>&1; echo "rc=$?" >> gpurun_out/r26_mn.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r26_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/r26_gputest.log
timeout 600 python tools/step_jitter.py 6 > gpurun_out/r26_jit.txt 2>&1
FQB_OZ_QMN=0 timeout 600 python tools/step_jitter.py 6 > gpurun_out/r26_jit_qmn0.txt 2>&1
