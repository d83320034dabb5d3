set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ozaki.py -q -x -p no:cacheprovider > gpurun_out/r5_oztest.log 2>&1; echo "rc=$?" >> gpurun_out/r5_oztest.log
timeout 900 python tools/ozaki_ab.py "FQB_OZ_S56=0" "FQB_OZ_S56=1" "FQB_OZ_S56=0" "FQB_OZ_S56=1" > gpurun_out/r5_ab.txt 2>&1
AB_SHAPE=8000,8000,50 timeout 600 python tools/ozaki_ab.py "FQB_OZ_S56=0" "FQB_OZ_S56=1" "FQB_OZ_S56=0" "FQB_OZ_S56=1" >> gpurun_out/r5_ab.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r5_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/r5_gputest.log
