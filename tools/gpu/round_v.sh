set -x
mkdir -p gpurun_out
timeout 600 python tools/ozaki_ab.py "FQB_OZ_WIDE=0" "FQB_OZ_WIDE=1" "FQB_OZ_WIDE=1 FQB_OZ_DIAGS=7" "FQB_OZ_WIDE=0" "FQB_OZ_WIDE=1" "FQB_OZ_WIDE=1 FQB_OZ_DIAGS=7" > gpurun_out/r23_ab.txt 2>&1
FQB_OZ_WIDE=1 timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_bigcases.py -q -p no:cacheprovider > gpurun_out/r23_tests_wide.log 2>&1; echo "rc=$?" >> gpurun_out/r23_tests_wide.log
FQB_OZ_WIDE=1 timeout 900 python tools/ozaki_accuracy.py > gpurun_out/r23_acc8w.txt 2>&1
FQB_OZ_WIDE=1 timeout 600 python tools/step_jitter.py 6 > gpurun_out/r23_jit8w.txt 2>&1
FQB_OZ_WIDE=1 FQB_OZ_DIAGS=7 timeout 600 python tools/step_jitter.py 6 > gpurun_out/r23_jit7w.txt 2>&1
