# one ncu --set full capture of k_search (3rd launch) for a config, after the same command ran clean
mkdir -p gpurun_out
c=${1:-C1}; shift
CMD="python bench.py --config $c $* --steps 2 --warmup 3 --no-cpu-baseline"
KNNG_PROFILE=1 timeout 900 $CMD > gpurun_out/ncu_plain_$c.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_search -s 3 -c 1 -f -o gpurun_out/k1_$c $CMD > gpurun_out/ncu_full_$c.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_full_$c.log
