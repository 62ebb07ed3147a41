# B = 1: the next insert's key-table row staged by the idle warps (double buffer): B = 1 parity, C0 timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sequential or batches_of_one or C0" > gpurun_out/r3n_par.log 2>&1; echo "rc=$?" >> gpurun_out/r3n_par.log
timeout 600 python -m pytest tests/test_gpu_strings.py tests/test_gpu_fullsize.py -q -x -k "sequential or C0_full" > gpurun_out/r3n_par2.log 2>&1; echo "rc=$?" >> gpurun_out/r3n_par2.log
if grep -q "rc=0" gpurun_out/r3n_par.log; then
  timeout 300 python scripts/prof_c0.py > gpurun_out/r3n_c0.log 2>&1
  timeout 600 python bench.py --config C0 --steps 20 --warmup 3 > gpurun_out/r3n_bench_C0.json 2> gpurun_out/r3n_bench_C0.err
fi
