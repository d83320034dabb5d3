# warm per-kernel breakdown of the C4 step (incl. cuSOLVER) + ncu of k_ozaki<true,7> at C4
set -x
mkdir -p gpurun_out
timeout 600 python tools/kernel_profile.py --config c4 --svd --runs 2 > gpurun_out/r3_kprof_c4.txt 2>&1
timeout 300 python tools/ozaki_c4_once.py tn 2 > gpurun_out/r3_oz_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k k_ozaki -s 1 -c 1 -o gpurun_out/r3_ozaki_c4 python tools/ozaki_c4_once.py tn 2 > gpurun_out/r3_ncu_oz.log 2>&1
