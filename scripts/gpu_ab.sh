# A/B of two builds of the library on the same K1 sweep: $1 = alternative .so (in paper_1602_06819_b200/), rest = configs
mkdir -p gpurun_out
alt=$1; shift
for spec in "$@"; do
  c=${spec%%:*}; extra=""; [ "$spec" != "$c" ] && extra=${spec#*:}
  tag=$(echo "$c$extra" | tr -c 'A-Za-z0-9_\n' '_' | cut -c1-60)
  timeout 900 python scripts/sweep_search.py $c $extra --settings plan > gpurun_out/ab_B_$tag.log 2>&1
  KNNG_LIB=$PWD/paper_1602_06819_b200/$alt timeout 900 python scripts/sweep_search.py $c $extra --settings plan > gpurun_out/ab_A_$tag.log 2>&1
done
