set -x
mkdir -p gpurun_out
timeout 600 python tools/ozaki_c4_once.py nn 2 > gpurun_out/r3b_once.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k k_ozaki --launch-skip 1 --launch-count 1 -o gpurun_out/r3b_ncu_nn python tools/ozaki_c4_once.py nn 2 > gpurun_out/r3b_ncu_nn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k k_ozaki --launch-skip 1 --launch-count 1 -o gpurun_out/r3b_ncu_tn python tools/ozaki_c4_once.py tn 2 > gpurun_out/r3b_ncu_tn.log 2>&1
FQB_PROFILE_RUNS=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3b_launches.csv python tools/profile_run.py > gpurun_out/r3b_launches.log 2>&1; echo "rc=$?" >> gpurun_out/r3b_launches.log
