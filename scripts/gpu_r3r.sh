# K1 launch bounds with the bulk-copy gathers: 6 CTAs/SM (80 regs, current) vs 7 (72) vs 5 (96); C3 8M, C2, C3 2M
mkdir -p gpurun_out
L=$PWD/paper_1602_06819_b200
for lib in libknng libknng_mb7 libknng_mb5; do
  KNNG_LIB=$L/$lib.so timeout 600 python scripts/k1_ab.py --config C2 --n0 1000000 --reps 3 - >> gpurun_out/r3r_${lib}_C2.log 2>&1
  KNNG_LIB=$L/$lib.so timeout 600 python scripts/k1_ab.py --config C3 --n0 2000000 --reps 3 - >> gpurun_out/r3r_${lib}_C3_2M.log 2>&1
done
for lib in libknng libknng_mb7; do
  KNNG_LIB=$L/$lib.so timeout 900 python scripts/k1_ab.py --config C3 --n0 8000000 --reps 3 - >> gpurun_out/r3r_${lib}_C3_8M.log 2>&1
done
