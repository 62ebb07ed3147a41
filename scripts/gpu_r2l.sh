mkdir -p gpurun_out
KNNG_LIB=$PWD/paper_1602_06819_b200/libknng_prof.so KNNG_PROFILE=1 timeout 300 python bench.py --config C0 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2l_bench_C0_prof.json 2> gpurun_out/r2l_bench_C0_prof.err
KNNG_NO_KT=1 KNNG_LIB=$PWD/paper_1602_06819_b200/libknng_prof.so KNNG_PROFILE=1 timeout 300 python bench.py --config C0 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2l_bench_C0_prof_nokt.json 2> gpurun_out/r2l_bench_C0_prof_nokt.err
KNNG_LIB=$PWD/paper_1602_06819_b200/libknng_prof.so KNNG_PROFILE=1 timeout 300 python scripts/k1_ab.py --config C1 --n0 100000 --reps 1 - > gpurun_out/r2l_prof_C1.log 2>&1
KNNG_LIB=$PWD/paper_1602_06819_b200/libknng_prof.so KNNG_PROFILE=1 timeout 300 python scripts/k1_ab.py --config C3 --n0 2000000 --reps 1 - > gpurun_out/r2l_prof_C3.log 2>&1
