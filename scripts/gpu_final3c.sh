# ncu refresh of K1 on C2 for the permutation-draw tree (launch list + one --set full capture)
mkdir -p gpurun_out/profiles_out
bash scripts/gpu_prof.sh C2
PROFILES_OUT=gpurun_out/profiles_out python scripts/summarize_profiles.py round2perm C2 gpurun_out/launches_C2.csv gpurun_out/prof_search_C2.ncu-rep > gpurun_out/f3_summ_C2.log 2>&1
python scripts/ncu_lines.py gpurun_out/prof_search_C2.ncu-rep 40 > gpurun_out/profiles_out/round2perm_C2_k_search_lines.txt 2>&1
rm -f gpurun_out/prof_search_C2.ncu-rep; gzip -f gpurun_out/launches_C2.csv
timeout 300 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/f3c_bench_C2.json 2> gpurun_out/f3c_bench_C2.err
