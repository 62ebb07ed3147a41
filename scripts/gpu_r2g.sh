mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/r2g_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_pytest.log
for spec in "C3 2000000" "C1 100000" "C2 1000000" "C4 500000"; do set -- $spec
  timeout 600 python scripts/k1_ab.py --config $1 --n0 $2 --reps 3 - KNNG_ROW_PF=1 > gpurun_out/r2g_ab_$1.log 2>&1
done
KNNG_LIB=$PWD/paper_1602_06819_b200/libknng_prof.so KNNG_PROFILE=1 timeout 600 python scripts/k1_ab.py --config C3 --n0 2000000 --reps 1 - KNNG_ROW_PF=1 > gpurun_out/r2g_prof_C3.log 2>&1
timeout 300 python bench.py --config C0 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/r2g_bench_C0.json 2> gpurun_out/r2g_bench_C0.err
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_search -c 1 -f -o gpurun_out/k1v4_C3 python scripts/k1_ab.py --config C3 --n0 2000000 --reps 1 > gpurun_out/r2g_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r2g_ncu.log
