set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r6a_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/r6a_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r6a_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r6a_smoke.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r6a_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r6a_bench_ref.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r6a_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r6a_bench.log
tail -3 gpurun_out/r6a_gputest.log; tail -2 gpurun_out/r6a_smoke.log; tail -c 600 gpurun_out/r6a_bench.log
