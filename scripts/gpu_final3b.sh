# closing lines of the permutation-draw tree for the remaining bench configs + the reference arm
mkdir -p gpurun_out
timeout 500 python bench.py --config C3 --n0 2000000 --steps 5 --warmup 3 --kmedoids-iters 3 --no-cpu-baseline > gpurun_out/f3_bench_C3_2M.json 2> gpurun_out/f3_bench_C3_2M.err
for c in S1 S2; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/f3_bench_$c.json 2> gpurun_out/f3_bench_$c.err
done
timeout 500 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/f3_ref.json 2> gpurun_out/f3_ref.err; echo "ref rc=$?" >> gpurun_out/f3_ref.err
