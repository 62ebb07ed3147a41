mkdir -p gpurun_out
L=$PWD/paper_1602_06819_b200
for lib in libknng libknng_mb7 libknng_mb8; do
  KNNG_LIB=$L/$lib.so timeout 600 python scripts/k1_ab.py --config C3 --n0 2000000 --reps 3 - > gpurun_out/r2m_${lib}_C3.log 2>&1
done
KNNG_LIB=$L/libknng_prof.so KNNG_PROFILE=1 timeout 300 python bench.py --config C0 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2m_bench_C0_prof.json 2> gpurun_out/r2m_bench_C0_prof.err
timeout 300 python bench.py --config C0 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/r2m_bench_C0.json 2> gpurun_out/r2m_bench_C0.err
timeout 300 python scripts/k1_ab.py --config C1 --n0 100000 --reps 3 - > gpurun_out/r2m_C1.log 2>&1
