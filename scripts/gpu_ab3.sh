mkdir -p gpurun_out
timeout 600 python scripts/k1_ab.py --config C3 --n0 2000000 --reps 2 - KNNG_GRID=444 KNNG_GRID=740 > gpurun_out/ab4_C3.log 2>&1
KNNG_LIB=$PWD/paper_1602_06819_b200/libknng_hack.so timeout 600 python scripts/k1_ab.py --config C3 --n0 2000000 --reps 2 - KNNG_GRID=444 > gpurun_out/ab4_C3_hack.log 2>&1
