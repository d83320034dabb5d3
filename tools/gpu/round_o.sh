set -x
mkdir -p gpurun_out
FQB_HOST_STATS=1 FQB_ALLOC_STATS=1 timeout 900 python tools/e2e_probe.py 3 > gpurun_out/r15_e2e.txt 2>&1
timeout 300 python tools/ozaki_c4_once.py tn 2 > gpurun_out/r15_oz_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k k_ozaki -s 1 -c 1 -o gpurun_out/r15_ozaki_c4 python tools/ozaki_c4_once.py tn 2 > gpurun_out/r15_ncu_oz.log 2>&1
timeout 300 python tools/sketch_sweep.py > gpurun_out/r15_sk_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --kernel-name-base function -k k_gather_spmm -s 40 -c 1 -o gpurun_out/r15_spmm_c3 python tools/sketch_sweep.py > gpurun_out/r15_ncu_sk.log 2>&1
timeout 300 python tools/profile_run.py > gpurun_out/r15_profile_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r15_launches.csv python tools/profile_run.py > gpurun_out/r15_ncu_launch.log 2>&1
