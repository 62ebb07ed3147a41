# ncu refresh of K1 on C1 for the permutation-draw tree (launch list + one --set full capture)
mkdir -p gpurun_out/profiles_out
bash scripts/gpu_prof.sh C1
PROFILES_OUT=gpurun_out/profiles_out python scripts/summarize_profiles.py round2perm C1 gpurun_out/launches_C1.csv gpurun_out/prof_search_C1.ncu-rep > gpurun_out/f3_summ_C1.log 2>&1
python scripts/ncu_lines.py gpurun_out/prof_search_C1.ncu-rep 40 > gpurun_out/profiles_out/round2perm_C1_k_search_lines.txt 2>&1
rm -f gpurun_out/prof_search_C1.ncu-rep; gzip -f gpurun_out/launches_C1.csv
