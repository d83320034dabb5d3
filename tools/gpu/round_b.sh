# GPU tests (new parity cases) + ncu of the dominant kernel at C4 and of the sparse sketch
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "graded or usv or bigcases or zeta" > gpurun_out/r2_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest.log
timeout 300 python tools/ozaki_c4_once.py tn 2 > gpurun_out/r2_oz_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ozaki -s 1 -c 1 -o gpurun_out/r2_ozaki_c4 python tools/ozaki_c4_once.py tn 2 > gpurun_out/r2_ncu_oz.log 2>&1
timeout 300 python tools/profile_run.py > gpurun_out/r2_profile_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv python tools/profile_run.py > gpurun_out/r2_ncu_launch.log 2>&1
