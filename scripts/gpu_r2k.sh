mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x --timeout 600 -k "fast_path or C0 or edge or forced or long_walk" > gpurun_out/r2k_pytest0.log 2>&1; echo "rc=$?" >> gpurun_out/r2k_pytest0.log
KNNG_LIB=$PWD/paper_1602_06819_b200/libknng_prof.so KNNG_PROFILE=1 timeout 300 python bench.py --config C0 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2k_bench_C0_prof.json 2> gpurun_out/r2k_bench_C0_prof.err
KNNG_LIB=$PWD/paper_1602_06819_b200/libknng_prof.so KNNG_PROFILE=1 timeout 300 python scripts/k1_ab.py --config C1 --n0 100000 --reps 1 - > gpurun_out/r2k_prof_C1.log 2>&1
timeout 300 python bench.py --config C0 --steps 100 --warmup 5 > gpurun_out/r2k_bench_C0.json 2> gpurun_out/r2k_bench_C0.err
timeout 600 python scripts/k1_ab.py --config C1 --n0 100000 --reps 3 - KNNG_XSMEM=0 KNNG_ESMEM=0 > gpurun_out/r2k_ab_C1.log 2>&1
