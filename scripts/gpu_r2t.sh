mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "sequential or fast_path or C0 or edge" > gpurun_out/r2t_pytest0.log 2>&1; echo "rc=$?" >> gpurun_out/r2t_pytest0.log
timeout 300 python bench.py --config C0 --steps 20 --warmup 3 > gpurun_out/r2t_bench_C0.json 2> gpurun_out/r2t_bench_C0.err
KNNG_LIB=$PWD/paper_1602_06819_b200/libknng_prof.so KNNG_PROFILE=1 timeout 300 python bench.py --config C0 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2t_bench_C0_prof.json 2> gpurun_out/r2t_bench_C0_prof.err
