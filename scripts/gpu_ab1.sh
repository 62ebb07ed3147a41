mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -rf --timeout 300 -k "not full_prefix and not C0_full" > gpurun_out/ab1_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab1_pytest.log
timeout 600 python scripts/k1_ab.py --config C3 --n0 2000000 --reps 2 - > gpurun_out/ab9_C3.log 2>&1
timeout 900 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab9_benchC3.log 2>&1
