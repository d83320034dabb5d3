set -x
mkdir -p gpurun_out
FQB_EIG_DEBUG=1 timeout 600 python tools/eig_time.py 500 --profile > gpurun_out/r18_eigprof.txt 2>&1
FQB_EIG_DEBUG=1 timeout 900 python tools/eig_time.py 2000 >> gpurun_out/r18_eigprof.txt 2>&1
