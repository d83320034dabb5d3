set -x
mkdir -p gpurun_out
( time timeout 1500 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/r6b_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r6b_bench_ref.log
( time timeout 1500 python3 bench.py --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/r6b_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r6b_bench.log
( time timeout 900 python3 bench.py ) > gpurun_out/r6b_bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/r6b_bench_default.log
tail -6 gpurun_out/r6b_bench_ref.log | cut -c1-300; tail -6 gpurun_out/r6b_bench.log | cut -c1-300; tail -6 gpurun_out/r6b_bench_default.log | cut -c1-300
