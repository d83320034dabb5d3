set -x
mkdir -p gpurun_out
timeout 900 python tools/ozaki_accuracy.py > gpurun_out/r22_acc8.txt 2>&1
FQB_OZ_DIAGS=7 timeout 900 python tools/ozaki_accuracy.py > gpurun_out/r22_acc7.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r22_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/r22_gputest.log
