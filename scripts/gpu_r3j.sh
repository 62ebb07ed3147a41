# round-2 closing measurement (session 3, final code: bulk-copy gathers): smoke, the full GPU suite, the
# default bench line (C3, with the CPU baseline), the launch list + one ncu --set full capture of K1 on C3
# (summarised on the box), the other configs' lines.  Only small files come back.
mkdir -p gpurun_out/profiles_out
nproc > gpurun_out/f4_nproc.txt; nvidia-smi > gpurun_out/f4_nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f4_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f4_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f4_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f4_pytest.log
timeout 1200 python bench.py > gpurun_out/f4_bench.json 2> gpurun_out/f4_bench.err; echo "bench rc=$?" >> gpurun_out/f4_bench.err
bash scripts/gpu_prof.sh C3
PROFILES_OUT=gpurun_out/profiles_out python scripts/summarize_profiles.py round2s4 C3 gpurun_out/launches_C3.csv gpurun_out/prof_search_C3.ncu-rep > gpurun_out/f4_summ_C3.log 2>&1
python scripts/ncu_lines.py gpurun_out/prof_search_C3.ncu-rep 40 > gpurun_out/profiles_out/round2s4_C3_k_search_lines.txt 2>&1
rm -f gpurun_out/prof_search_C3.ncu-rep; gzip -f gpurun_out/launches_C3.csv
timeout 600 python bench.py --config C0 --steps 20 --warmup 3 > gpurun_out/f4_bench_C0.json 2> gpurun_out/f4_bench_C0.err
for c in C1 C2 C4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/f4_bench_$c.json 2> gpurun_out/f4_bench_$c.err
done
timeout 900 python bench.py --config C3 --n0 2000000 --steps 5 --warmup 3 --kmedoids-iters 3 --no-cpu-baseline > gpurun_out/f4_bench_C3_2M.json 2> gpurun_out/f4_bench_C3_2M.err
du -sh gpurun_out
for c in S1 S2; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/f4_bench_$c.json 2> gpurun_out/f4_bench_$c.err
done
