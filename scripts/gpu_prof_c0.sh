# C0 (B = 1 sequential launch): one ncu --set full capture of the fused k_search with source lines
mkdir -p gpurun_out
timeout 300 python scripts/prof_c0.py > gpurun_out/r3h_c0_plain.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_search -s 3 -c 1 -f -o gpurun_out/prof_c0 python scripts/prof_c0.py > gpurun_out/r3h_ncu.log 2>&1
python scripts/ncu_lines.py gpurun_out/prof_c0.ncu-rep 60 > gpurun_out/r3h_c0_lines.txt 2>&1
rm -f gpurun_out/prof_c0.ncu-rep
