# K1 bulk-copy (TMA) gathers: forced-path parity (bulk vs oracle), then the A/B (KNNG_BULK=0 vs 1) on C3 8M, C2, C3 2M
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "bulk or long_walks" > gpurun_out/r3g_par.log 2>&1; echo "rc=$?" >> gpurun_out/r3g_par.log
if grep -q "rc=0" gpurun_out/r3g_par.log; then
  timeout 900 python scripts/k1_ab.py --config C3 --n0 8000000 --reps 3 KNNG_BULK=0 KNNG_BULK=1 KNNG_BULK=0 KNNG_BULK=1 > gpurun_out/r3g_C3_8M.log 2>&1
  timeout 600 python scripts/k1_ab.py --config C2 --n0 1000000 --reps 3 KNNG_BULK=0 KNNG_BULK=1 KNNG_BULK=0 KNNG_BULK=1 > gpurun_out/r3g_C2.log 2>&1
  timeout 600 python scripts/k1_ab.py --config C3 --n0 2000000 --reps 3 KNNG_BULK=0 KNNG_BULK=1 > gpurun_out/r3g_C3_2M.log 2>&1
fi
# register-mask JW evaluator: string parity + the S1 line
timeout 900 python -m pytest tests/test_gpu_strings.py -q -x > gpurun_out/r3g_strings.log 2>&1; echo "rc=$?" >> gpurun_out/r3g_strings.log
timeout 600 python bench.py --config S1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r3g_bench_S1.json 2> gpurun_out/r3g_bench_S1.err
timeout 600 python bench.py --config S2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r3g_bench_S2.json 2> gpurun_out/r3g_bench_S2.err
