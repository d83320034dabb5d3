set -x
mkdir -p gpurun_out
timeout 600 python tools/ozaki_ab.py "FQB_OZ_DIAGS=8" "FQB_OZ_DIAGS=7" "FQB_OZ_DIAGS=8" "FQB_OZ_DIAGS=7" > gpurun_out/r21_ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_bigcases.py -q -p no:cacheprovider > gpurun_out/r21_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r21_tests.log
FQB_OZ_DIAGS=7 timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_bigcases.py tests/test_gpu_fullsize.py -q -p no:cacheprovider > gpurun_out/r21_tests_d7.log 2>&1; echo "rc=$?" >> gpurun_out/r21_tests_d7.log
timeout 600 python tools/step_jitter.py 6 > gpurun_out/r21_jit8.txt 2>&1
FQB_OZ_DIAGS=7 timeout 600 python tools/step_jitter.py 6 > gpurun_out/r21_jit7.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r21_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r21_bench.log
