# parity suite + the lines of the configs a change touches (CONFIGS="C4 ..." in the env)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/k_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/k_pytest_gpu.log
for c in $CONFIGS; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/k_bench_$c.json 2> gpurun_out/k_bench_$c.err
done
