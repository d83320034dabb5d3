mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bigcases.py tests/test_gpu_fullsize.py tests/test_gpu_multirank.py tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/r3d_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3d_tests.log
for v in 0 1 0 1; do echo "FQB_OZ_B=$v"; FQB_OZ_B=$v timeout 600 python tools/step_jitter.py 4; done > gpurun_out/r3d_jit.txt 2>&1
