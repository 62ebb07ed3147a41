# K1 window refresh from the walk's list: parity on the forced plan paths / long walks / streams, then the
# K1 A/B (previous library vs new) on C3 8M, C2 1M, C4 500k
mkdir -p gpurun_out
L=$PWD/paper_1602_06819_b200
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -k "forced or long_walks or C3_full or C2_full" > gpurun_out/r3e_par.log 2>&1; echo "rc=$?" >> gpurun_out/r3e_par.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "search or stream or insert or partition" > gpurun_out/r3e_par2.log 2>&1; echo "rc=$?" >> gpurun_out/r3e_par2.log
for lib in libknng_prev libknng; do
  KNNG_LIB=$L/$lib.so timeout 900 python scripts/k1_ab.py --config C3 --n0 8000000 --reps 3 - > gpurun_out/r3e_${lib}_C3_8M.log 2>&1
  KNNG_LIB=$L/$lib.so timeout 900 python scripts/k1_ab.py --config C2 --n0 1000000 --reps 3 - > gpurun_out/r3e_${lib}_C2.log 2>&1
  KNNG_LIB=$L/$lib.so timeout 900 python scripts/k1_ab.py --config C4 --n0 500000 --reps 3 - > gpurun_out/r3e_${lib}_C4.log 2>&1
done
