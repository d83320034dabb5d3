mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tsmm.py tests/test_gpu_parity.py tests/test_gpu_bigcases.py tests/test_gpu_edge_parity.py tests/test_gpu_fp32.py tests/test_gpu_multirank.py tests/test_gpu_int8_bgs.py tests/test_gpu_fixed_rank_device.py -q -p no:cacheprovider -x > gpurun_out/r3m_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3m_tests.log
timeout 300 python tools/tsmm_once.py > gpurun_out/r3m_once.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_ts_ --log-file gpurun_out/r3m_ts_launches.csv python tools/tsmm_once.py > gpurun_out/r3m_ncu.log 2>&1
