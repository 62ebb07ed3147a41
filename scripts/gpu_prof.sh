# profiling pass for one config: a clean bench line, the launch list (all kernels, device times)
# and one ncu --set full capture of k_search; each ncu command only after the same command ran clean.
# usage: bash scripts/gpu_prof.sh C1 [extra bench args]
mkdir -p gpurun_out
c=${1:-C1}; shift
CMD="python bench.py --config $c $* --steps 2 --warmup 3 --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/prof_plain_$c.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv $CMD > gpurun_out/ncu_launches_$c.log 2>&1
echo "launches rc=$?" >> gpurun_out/ncu_launches_$c.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_search -s 3 -c 1 -f -o gpurun_out/prof_search_$c $CMD > gpurun_out/ncu_full_$c.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_full_$c.log
