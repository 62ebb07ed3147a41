mkdir -p gpurun_out
KNNG_PROFILE=1 timeout 900 python bench.py --config C2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/kp_C2.log 2>&1
KNNG_PROFILE=1 timeout 900 python bench.py --config C3 --n0 2000000 --steps 2 --warmup 3 --kmedoids-iters 2 --no-cpu-baseline > gpurun_out/kp_C3.log 2>&1
