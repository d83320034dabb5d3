# 56-row Z slices (default) vs FQB_OZ_ZR=64: GPU tests, bench A/B, config 3/4 times
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_fp32.py -x -q > gpurun_out/zr_tests.log 2>&1; echo "rc=$?" >> gpurun_out/zr_tests.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/zr_gpu_all.log 2>&1; echo "rc=$?" >> gpurun_out/zr_gpu_all.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/zr_bench56.json 2>/dev/null
FQB_OZ_ZR=64 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/zr_bench64.json 2>/dev/null
timeout 400 python tools/config_time.py c4 > gpurun_out/zr_c4_56.txt 2>&1
FQB_OZ_ZR=64 timeout 400 python tools/config_time.py c4 > gpurun_out/zr_c4_64.txt 2>&1
timeout 300 python tools/config_time.py c3 > gpurun_out/zr_c3_56.txt 2>&1
echo done
