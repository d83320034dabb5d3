set -x
mkdir -p gpurun_out
FQB_ALLOC_STATS=1 FQB_HOST_STATS=1 timeout 900 python tools/step_jitter.py 5 > gpurun_out/r9_alloc.txt 2>&1
