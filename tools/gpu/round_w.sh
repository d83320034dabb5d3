set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ozaki_variants.py tests/test_gpu_ozaki.py -q -p no:cacheprovider > gpurun_out/r24_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r24_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r24_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r24_bench.log
timeout 600 python tools/ozaki_c4_once.py nn 2 > gpurun_out/r24_once.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k k_ozaki --launch-skip 1 --launch-count 1 -o gpurun_out/r24_ncu_nn python tools/ozaki_c4_once.py nn 2 > gpurun_out/r24_ncu_nn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k k_ozaki --launch-skip 1 --launch-count 1 -o gpurun_out/r24_ncu_tn python tools/ozaki_c4_once.py tn 2 > gpurun_out/r24_ncu_tn.log 2>&1
