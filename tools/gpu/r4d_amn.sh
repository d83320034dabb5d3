mkdir -p gpurun_out
for l in 500 1000 1900; do timeout 300 python tools/amn_once.py $l 5; done > gpurun_out/r4d_amn.txt 2>&1
timeout 300 python tools/amn_once.py 1000 2 > gpurun_out/r4d_once.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k k_ozaki --launch-skip 1 --launch-count 1 -o gpurun_out/r4d_ncu_amn python tools/amn_once.py 1000 2 > gpurun_out/r4d_ncu.log 2>&1
