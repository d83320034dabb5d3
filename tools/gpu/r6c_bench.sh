set -x
mkdir -p gpurun_out
( time timeout 1500 python3 bench.py --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/r6c_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r6c_bench.log
tail -6 gpurun_out/r6c_bench.log | cut -c1-300
