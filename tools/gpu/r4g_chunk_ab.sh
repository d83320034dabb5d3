mkdir -p gpurun_out
timeout 900 python tools/ozaki_ab.py "FQB_OZ_CHUNK=256" "FQB_OZ_CHUNK=336" "FQB_OZ_CHUNK=256" "FQB_OZ_CHUNK=336" > gpurun_out/r4g_ab.txt 2>&1
for v in 256 336 256 336; do echo "FQB_OZ_CHUNK=$v"; FQB_OZ_CHUNK=$v timeout 600 python tools/step_jitter.py 3; done > gpurun_out/r4g_jit.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_bigcases.py -q -p no:cacheprovider -x > gpurun_out/r4g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r4g_tests.log
