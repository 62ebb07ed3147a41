# ncu --set full of the tcgen05 exact-build kernels (u8: C1's graph_init; f32: a 200k-point C2-shaped
# graph_init), summarised on the box (tensor-pipe and memory metrics), reports deleted
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on -k regex:k_tc_topk_u8 -c 1 -f -o gpurun_out/tc_u8 python scripts/time_build.py C1 --no-simt > gpurun_out/ncu_tc_u8.log 2>&1
timeout 900 ncu --set full --import-source on -k regex:k_tc_topk_f32 -c 1 -f -o gpurun_out/tc_f32 python scripts/time_build.py C2 --n0 200000 --no-simt > gpurun_out/ncu_tc_f32.log 2>&1
for r in tc_u8 tc_f32; do
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
  python scripts/ncu_lines.py gpurun_out/$r.ncu-rep 25 > gpurun_out/${r}_lines.txt 2>&1
  rm -f gpurun_out/$r.ncu-rep
done
