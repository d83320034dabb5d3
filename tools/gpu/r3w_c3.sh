mkdir -p gpurun_out
FQB_PROFILE=1 timeout 900 python tools/config_time.py c3 > gpurun_out/r3w_c3.txt 2>&1
