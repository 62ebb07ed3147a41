mkdir -p gpurun_out
for v in libknng.so libknng_b.so; do
  echo "== $v" >> gpurun_out/ab.log
  KNNG_LIB=$PWD/paper_1602_06819_b200/$v KNNG_PROFILE=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline >> gpurun_out/ab.log 2>&1
done
