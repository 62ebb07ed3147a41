mkdir -p gpurun_out
KNNG_PROFILE=1 timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/kprof.log 2>&1
echo "rc=$?" >> gpurun_out/kprof.log
