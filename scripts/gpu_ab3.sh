mkdir -p gpurun_out
KNNG_LIB=$PWD/paper_1602_06819_b200/libknng_mb7.so KNNG_PROFILE=1 timeout 600 python scripts/k1_ab.py --config C3 --n0 2000000 --reps 2 - > gpurun_out/ab8_C3_mb7.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_search -c 1 -f -o gpurun_out/k1v3b_C3 python scripts/k1_ab.py --config C3 --n0 2000000 --reps 1 > gpurun_out/ncuv3b.log 2>&1
echo "rc=$?" >> gpurun_out/ncuv3b.log
