mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x --timeout 600 -k "jaccard or C4" > gpurun_out/r2s_pytest0.log 2>&1; echo "rc=$?" >> gpurun_out/r2s_pytest0.log
timeout 600 python scripts/k1_ab.py --config C4 --n0 500000 --reps 3 - > gpurun_out/r2s_C4.log 2>&1
timeout 900 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2s_bench_C4.json 2> gpurun_out/r2s_bench_C4.err
timeout 300 python scripts/k1_ab.py --config C3 --n0 2000000 --reps 3 - > gpurun_out/r2s_C3.log 2>&1
