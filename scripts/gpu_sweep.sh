mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 600 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for spec in "$@"; do
  c=${spec%%:*}; extra=""; [ "$spec" != "$c" ] && extra=${spec#*:}
  tag=$(echo "$c$extra" | tr -c 'A-Za-z0-9_\n' '_' | cut -c1-60)
  timeout 900 python scripts/sweep_search.py $c $extra > gpurun_out/sw_$tag.log 2>&1; echo "rc=$?" >> gpurun_out/sw_$tag.log
done
