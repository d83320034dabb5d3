set -x
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/r6e_launches_bench.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r6e_ncu_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r6e_ncu_bench.log
tail -3 gpurun_out/r6e_ncu_bench.log | cut -c1-300; wc -l gpurun_out/r6e_launches_bench.csv
