# bench lines for the other BASELINE.json configs (not the driver's bench line: C1 is the metric's workload)
mkdir -p gpurun_out
for c in C0 C2 C4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$c.log
done
timeout 900 python bench.py --config C3 --n0 2000000 --steps 5 --warmup 3 --kmedoids-iters 3 --no-cpu-baseline > gpurun_out/bench_C3_2M.log 2>&1; echo "rc=$?" >> gpurun_out/bench_C3_2M.log
