set -x
mkdir -p gpurun_out
timeout 900 python tools/ozaki_ab.py "FQB_OZ_L2HINT=0 FQB_OZ_BSTAGES=2" "FQB_OZ_L2HINT=1 FQB_OZ_BSTAGES=2" "FQB_OZ_L2HINT=0 FQB_OZ_BSTAGES=3" "FQB_OZ_L2HINT=1 FQB_OZ_BSTAGES=3" "FQB_OZ_L2HINT=0 FQB_OZ_BSTAGES=2" "FQB_OZ_L2HINT=1 FQB_OZ_BSTAGES=3" > gpurun_out/r4_ab.txt 2>&1
AB_SHAPE=8000,8000,50 timeout 600 python tools/ozaki_ab.py "FQB_OZ_L2HINT=0" "FQB_OZ_L2HINT=1" "FQB_OZ_L2HINT=1 FQB_OZ_BSTAGES=3" >> gpurun_out/r4_ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_ozaki.py -q -p no:cacheprovider > gpurun_out/r4_oztest.log 2>&1; echo "rc=$?" >> gpurun_out/r4_oztest.log
