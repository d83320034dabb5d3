set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r14_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/r14_gputest.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r14_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r14_bench.log
