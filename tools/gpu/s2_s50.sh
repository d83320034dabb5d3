set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ozaki_variants.py -q -p no:cacheprovider -x > gpurun_out/s2_variants.log 2>&1; echo "rc=$?" >> gpurun_out/s2_variants.log
timeout 900 python -m pytest tests/test_gpu_ozaki.py -q -p no:cacheprovider -x > gpurun_out/s2_ozaki.log 2>&1; echo "rc=$?" >> gpurun_out/s2_ozaki.log
timeout 600 python tools/ozaki_ab.py "FQB_OZ_S50=0" "FQB_OZ_S50=1" "FQB_OZ_S50=0" "FQB_OZ_S50=1" > gpurun_out/s2_ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_bigcases.py -q -p no:cacheprovider -x > gpurun_out/s2_big.log 2>&1; echo "rc=$?" >> gpurun_out/s2_big.log
timeout 600 python tools/step_jitter.py 4 > gpurun_out/s2_jit.txt 2>&1
FQB_OZ_S50=0 timeout 600 python tools/step_jitter.py 4 > gpurun_out/s2_jit_s56.txt 2>&1
