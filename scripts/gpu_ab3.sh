mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_search -c 1 -f -o gpurun_out/k1v3_C3 python scripts/k1_ab.py --config C3 --n0 2000000 --reps 1 > gpurun_out/ncuv3.log 2>&1
echo "rc=$?" >> gpurun_out/ncuv3.log
