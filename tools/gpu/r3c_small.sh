mkdir -p gpurun_out
for l in 500 1000 1900; do timeout 300 python tools/small_gemm_c4.py $l; done > gpurun_out/r3c_small.txt 2>&1; echo "rc=$?" >> gpurun_out/r3c_small.txt
