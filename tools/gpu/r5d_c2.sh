set -x
mkdir -p gpurun_out
timeout 900 python bench.py --workload c2 --steps 10 --warmup 3 > gpurun_out/r5d_c2.log 2>&1; echo "rc=$?" >> gpurun_out/r5d_c2.log
timeout 900 python bench.py --workload c2 --impl reference --steps 2 --warmup 0 > gpurun_out/r5d_c2_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r5d_c2_ref.log
