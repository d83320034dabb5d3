set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r13_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/r13_gputest.log
for v in 0 512 1024 1536; do echo "QNN_MIN=$v"; FQB_OZ_QNN_MIN=$v timeout 600 python tools/step_jitter.py 3 2>&1 | grep step; done > gpurun_out/r13_ab.txt
