set -x
mkdir -p gpurun_out
FQB_EIG_DEBUG=1 timeout 900 python -m pytest tests/test_gpu_eig.py -q -p no:cacheprovider > gpurun_out/r19_eig.log 2>&1; echo "rc=$?" >> gpurun_out/r19_eig.log
FQB_EIG_DEBUG=1 timeout 600 python tools/eig_time.py 2000 --profile > gpurun_out/r19_eigprof.txt 2>&1
