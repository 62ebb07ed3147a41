# end-of-round measurement: smoke, GPU tests, the default bench line (with the CPU baseline), the
# other configs' lines, and the ncu launch list + full capture of K1 for C1 and C2.  The ncu
# reports are summarised on the box (gpurun_out/profiles_out/) and deleted: only small files return.
mkdir -p gpurun_out/profiles_out
bash scripts/gpu_round.sh
for c in C1 C2; do
  bash scripts/gpu_prof.sh $c
  PROFILES_OUT=gpurun_out/profiles_out python scripts/summarize_profiles.py round1 $c gpurun_out/launches_$c.csv gpurun_out/prof_search_$c.ncu-rep > gpurun_out/summ_$c.log 2>&1
  rm -f gpurun_out/prof_search_$c.ncu-rep
  gzip -f gpurun_out/launches_$c.csv
done
bash scripts/gpu_configs.sh
timeout 1500 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_C3.log
du -sh gpurun_out
