# bench lines of every config (no CPU baseline), each under its own timeout
mkdir -p gpurun_out
tag=${1:-r2c}
timeout 300 python bench.py --config C1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_C1.log 2>&1
timeout 400 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_C2.log 2>&1
timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_C3.log 2>&1
timeout 400 python bench.py --config C4 --n0 500000 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_C4_500k.log 2>&1
timeout 300 python bench.py --config C0 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_C0.log 2>&1
