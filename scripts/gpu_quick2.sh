mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 600 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b_C1.log 2>&1
timeout 900 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b_C2.log 2>&1
timeout 900 python bench.py --config C3 --n0 2000000 --steps 3 --warmup 3 --kmedoids-iters 3 --no-cpu-baseline > gpurun_out/b_C3.log 2>&1
