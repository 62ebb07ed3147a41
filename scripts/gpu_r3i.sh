# JW via the query's character position lists: string parity, then the S1 / S2 lines with the CPU baseline
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_strings.py -q -x > gpurun_out/r3i_strings.log 2>&1; echo "rc=$?" >> gpurun_out/r3i_strings.log
if grep -q "rc=0" gpurun_out/r3i_strings.log; then
  for c in S1 S2; do
    timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/r3i_bench_$c.json 2> gpurun_out/r3i_bench_$c.err
  done
fi
