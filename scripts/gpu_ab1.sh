mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -rf --timeout 300 -k "not full_prefix and not C0_full" > gpurun_out/ab1_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab1_pytest.log
export KNNG_LIB=$PWD/paper_1602_06819_b200/libknng_prof.so KNNG_PROFILE=1
timeout 900 python scripts/k1_ab.py --config C3 --n0 2000000 --reps 1 - KNNG_WALK_PREFETCH=0 KNNG_RING=8 KNNG_WALK_PREFETCH=0,KNNG_GRID=148 > gpurun_out/ab2_C3.log 2>&1; echo "rc=$?" >> gpurun_out/ab2_C3.log
timeout 900 python scripts/k1_ab.py --config C1 --n0 100000 --reps 2 - KNNG_WALK_PREFETCH=0 KNNG_RING=16 > gpurun_out/ab2_C1.log 2>&1; echo "rc=$?" >> gpurun_out/ab2_C1.log
