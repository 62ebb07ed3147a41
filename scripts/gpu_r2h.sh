mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/r2h_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2h_pytest.log
timeout 600 python scripts/k1_ab.py --config C1 --n0 100000 --reps 3 - KNNG_ESMEM=0 KNNG_NS2=0 > gpurun_out/r2h_ab_C1.log 2>&1
timeout 600 python scripts/k1_ab.py --config C3 --n0 2000000 --reps 3 - KNNG_ESMEM=1 > gpurun_out/r2h_ab_C3.log 2>&1
timeout 300 python scripts/k1_ab.py --config C0 --n0 2000 --nq 1 --reps 5 - KNNG_ESMEM=0 KNNG_NS2=0 > gpurun_out/r2h_ab_C0.log 2>&1
for c in C0 C1; do timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2h_bench_$c.json 2> gpurun_out/r2h_bench_$c.err; done
