set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r1_gpu.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r1_smoke.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r1_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r1_bench.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r1_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1_gputest.log
