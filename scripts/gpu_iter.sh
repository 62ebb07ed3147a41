# iteration run: GPU parity tests, then KNNG_PROFILE bench lines for the configs given as arguments
# (e.g. "C1" "C2" "C4:--n0 500000"); logs under gpurun_out/
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 600 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for spec in "$@"; do
  c=${spec%%:*}; extra=""; [ "$spec" != "$c" ] && extra=${spec#*:}
  tag=$(echo "$c$extra" | tr -c 'A-Za-z0-9_\n' '_' | cut -c1-60)
  KNNG_PROFILE=1 timeout 900 python bench.py --config $c $extra --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/it_$tag.log 2>&1
  echo "rc=$?" >> gpurun_out/it_$tag.log
done
