mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2f_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -rf -x --timeout 900 --durations=15 > gpurun_out/r2f_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_pytest.log
for c in C0 C1 C2; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2f_bench_$c.json 2> gpurun_out/r2f_bench_$c.err; done
for t in memcheck racecheck synccheck; do timeout 900 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize_case.py > gpurun_out/r2f_san_$t.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_san_$t.log; done
