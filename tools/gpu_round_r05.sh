set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_r05.json 2> gpurun_out/bench_r05.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref_r05.json 2>&1
timeout 300 python tools/kernel_profile.py --svd > gpurun_out/kernel_profile_c2_r05.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_bench_r05.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ozaki -s 30 -c 1 -o gpurun_out/ozaki_r05 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo done
