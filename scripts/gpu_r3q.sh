# K1 A/B: single-barrier bulk gathers (0085189) vs the two-barrier bookkeeping (current), C2 / C3 at 2M / C1
mkdir -p gpurun_out
L=$PWD/paper_1602_06819_b200
for lib in libknng_prev libknng libknng_prev libknng; do
  KNNG_LIB=$L/$lib.so timeout 600 python scripts/k1_ab.py --config C2 --n0 1000000 --reps 3 - >> gpurun_out/r3q_${lib}_C2.log 2>&1
  KNNG_LIB=$L/$lib.so timeout 600 python scripts/k1_ab.py --config C3 --n0 2000000 --reps 3 - >> gpurun_out/r3q_${lib}_C3_2M.log 2>&1
done
