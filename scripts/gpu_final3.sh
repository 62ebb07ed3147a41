# round-2 closing run on the permutation-draw tree (perm_e): smoke, the default bench line (C3, CPU
# baseline included), the launch list + one ncu --set full capture of K1 on C3 (summarised on the box;
# the pre-perm_e capture under profiles/ is stale), the GPU parity suite, the other configs' lines.
mkdir -p gpurun_out/profiles_out
nproc > gpurun_out/f3_nproc.txt; nvidia-smi > gpurun_out/f3_nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f3_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f3_smoke.log
timeout 1200 python bench.py > gpurun_out/f3_bench.json 2> gpurun_out/f3_bench.err; echo "bench rc=$?" >> gpurun_out/f3_bench.err
bash scripts/gpu_prof.sh C3
PROFILES_OUT=gpurun_out/profiles_out python scripts/summarize_profiles.py round2perm C3 gpurun_out/launches_C3.csv gpurun_out/prof_search_C3.ncu-rep > gpurun_out/f3_summ_C3.log 2>&1
python scripts/ncu_lines.py gpurun_out/prof_search_C3.ncu-rep 40 > gpurun_out/profiles_out/round2perm_C3_k_search_lines.txt 2>&1
rm -f gpurun_out/prof_search_C3.ncu-rep; gzip -f gpurun_out/launches_C3.csv
timeout 900 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/f3_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f3_pytest_gpu.log
timeout 300 python bench.py --config C0 --steps 20 --warmup 3 > gpurun_out/f3_bench_C0.json 2> gpurun_out/f3_bench_C0.err
for c in C2 C1 C4; do
  timeout 400 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/f3_bench_$c.json 2> gpurun_out/f3_bench_$c.err
done
du -sh gpurun_out
