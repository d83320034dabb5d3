set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r5a_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/r5a_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5a_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r5a_smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r5a_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r5a_bench.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r5a_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r5a_bench_ref.log
FQB_PROFILE_RUNS=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r5a_launches.csv python tools/profile_run.py > gpurun_out/r5a_launches.log 2>&1; echo "rc=$?" >> gpurun_out/r5a_launches.log
