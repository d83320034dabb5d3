mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tsmm.py -q -p no:cacheprovider -x > gpurun_out/r4j_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r4j_tests.log
timeout 300 python tools/tsmm_once.py > gpurun_out/r4j_once.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_ts_ --log-file gpurun_out/r4j_ts_launches.csv python tools/tsmm_once.py > gpurun_out/r4j_ncu.log 2>&1
