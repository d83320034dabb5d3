set -x
mkdir -p gpurun_out
FQB_EIG_DEBUG=1 timeout 900 python -m pytest tests/test_gpu_eig.py -q -x -p no:cacheprovider -k large > gpurun_out/r17_eig.log 2>&1; echo "rc=$?" >> gpurun_out/r17_eig.log
for n in 500 2000; do timeout 600 python tools/eig_time.py $n; done > gpurun_out/r17_eigtime.txt 2>&1
