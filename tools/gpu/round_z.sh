set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ozaki.py -q -p no:cacheprovider -k "mn" > gpurun_out/r27_mn.log 2>&1; echo "rc=$?" >> gpurun_out/r27_mn.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r27_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/r27_gputest.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r27_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r27_bench.log
