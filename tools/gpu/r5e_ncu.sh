set -x
mkdir -p gpurun_out
timeout 600 python tools/ozaki_c4_once.py tn 2 > gpurun_out/r5e_once.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k k_ozaki --launch-skip 1 --launch-count 1 -o gpurun_out/r5e_ncu_tn python tools/ozaki_c4_once.py tn 2 > gpurun_out/r5e_ncu_tn.log 2>&1
timeout 600 ncu --set full --clock-control none --kernel-name-base function -k k_ozaki --launch-skip 8 --launch-count 1 -o gpurun_out/r5e_ncu_c2 python bench.py --workload c2 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r5e_ncu_c2.log 2>&1
for f in tn c2; do ncu -i gpurun_out/r5e_ncu_$f.ncu-rep --page raw --csv > gpurun_out/r5e_ncu_${f}_raw.csv 2>/dev/null; done
echo done
