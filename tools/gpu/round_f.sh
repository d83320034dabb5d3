set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -x -p no:cacheprovider > gpurun_out/r6_multirank.log 2>&1; echo "rc=$?" >> gpurun_out/r6_multirank.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r6_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r6_bench.log
