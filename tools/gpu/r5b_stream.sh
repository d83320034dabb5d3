set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_host_stream.py tests/test_gpu_comm.py tests/test_gpu_edge_parity.py tests/test_gpu_fixed_rank_device.py tests/test_gpu_eig.py tests/test_gpu_multirank.py -q -p no:cacheprovider > gpurun_out/r5b_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r5b_tests.log
FQB_OUT_TAIL=1 timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r5b_bench_tail.log 2>&1; echo "rc=$?" >> gpurun_out/r5b_bench_tail.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r5b_bench_stream.log 2>&1; echo "rc=$?" >> gpurun_out/r5b_bench_stream.log
FQB_OUT_TAIL=1 timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r5b_bench_tail2.log 2>&1; echo "rc=$?" >> gpurun_out/r5b_bench_tail2.log
