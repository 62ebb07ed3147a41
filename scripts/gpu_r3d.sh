# string measures after the fused-path store-view fix: string parity, sequential Jaccard, then bench lines S1 / S2
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_strings.py -q > gpurun_out/r3d_strings.log 2>&1; echo "rc=$?" >> gpurun_out/r3d_strings.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "sequential or batches_of_one or jaccard" > gpurun_out/r3d_seq.log 2>&1; echo "rc=$?" >> gpurun_out/r3d_seq.log
for c in S1 S2; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/r3d_bench_$c.json 2> gpurun_out/r3d_bench_$c.err
done
