mkdir -p gpurun_out
L=$PWD/paper_1602_06819_b200
for lib in libknng libknng_l2h; do
  KNNG_LIB=$L/$lib.so timeout 600 python scripts/k1_ab.py --config C3 --n0 2000000 --reps 3 - > gpurun_out/r2u_${lib}_C3_2M.log 2>&1
  KNNG_LIB=$L/$lib.so timeout 600 python scripts/k1_ab.py --config C2 --n0 1000000 --reps 3 - > gpurun_out/r2u_${lib}_C2.log 2>&1
done
for lib in libknng libknng_l2h; do
  KNNG_LIB=$L/$lib.so timeout 900 python scripts/k1_ab.py --config C3 --n0 8000000 --reps 3 - > gpurun_out/r2u_${lib}_C3_8M.log 2>&1
done
