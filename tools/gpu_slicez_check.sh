# k_slice_z with all max-pass loads in flight: ozaki tests, whole GPU suite, warm kernel profile, bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_fp32.py -x -q > gpurun_out/sz_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sz_tests.log
timeout 300 python tools/kernel_profile.py --svd > gpurun_out/sz_profile.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/sz_gpu_all.log 2>&1; echo "rc=$?" >> gpurun_out/sz_gpu_all.log
timeout 600 python bench.py > gpurun_out/sz_bench.json 2> gpurun_out/sz_bench.err
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/sz_smoke.log 2>&1
echo done
