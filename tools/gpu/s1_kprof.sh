set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/s1_smi.txt 2>&1
timeout 900 python tools/kernel_profile.py --config c4 --svd --runs 2 > gpurun_out/s1_kprof_c4.txt 2>&1
timeout 600 python tools/kernel_profile.py --config c2 --svd --runs 5 > gpurun_out/s1_kprof_c2.txt 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/s1_bench.log 2>&1; echo "rc=$?" >> gpurun_out/s1_bench.log
