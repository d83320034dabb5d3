set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r3a_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/r3a_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3a_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r3a_smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r3a_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r3a_bench.log
timeout 900 python tools/kernel_profile.py --config c4 --svd --runs 2 > gpurun_out/r3a_kprof_c4.txt 2>&1
