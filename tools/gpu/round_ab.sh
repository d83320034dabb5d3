set -x
mkdir -p gpurun_out
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_ozaki.py -q -p no:cacheprovider -k "mn or pass_timing or again" > gpurun_out/r29_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/r29_memcheck.log
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_ozaki.py -q -p no:cacheprovider -k "mn_fp64_accuracy and 1000-200" > gpurun_out/r29_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/r29_racecheck.log
