# B = 1 with the rows in shared memory (srows): B = 1 / sequential parity, then C0 timing (srows vs KNNG_NO_SROWS)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sequential or batches_of_one or C0" > gpurun_out/r3l_par.log 2>&1; echo "rc=$?" >> gpurun_out/r3l_par.log
timeout 600 python -m pytest tests/test_gpu_strings.py -q -x -k "sequential" > gpurun_out/r3l_par2.log 2>&1; echo "rc=$?" >> gpurun_out/r3l_par2.log
if grep -q "rc=0" gpurun_out/r3l_par.log; then
  timeout 300 python scripts/prof_c0.py > gpurun_out/r3l_c0_srows.log 2>&1
  KNNG_NO_SROWS=1 timeout 300 python scripts/prof_c0.py > gpurun_out/r3l_c0_nosrows.log 2>&1
  timeout 600 python bench.py --config C0 --steps 20 --warmup 3 > gpurun_out/r3l_bench_C0.json 2> gpurun_out/r3l_bench_C0.err
fi
