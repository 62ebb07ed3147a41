# partition-local store: GPU tests, then K1 A/B (base library vs the new one) on C3 8M / C4 500k, and the bench line
mkdir -p gpurun_out
L=$PWD/paper_1602_06819_b200
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r3b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r3b_pytest.log
for lib in libknng_base libknng; do
  KNNG_LIB=$L/$lib.so timeout 900 python scripts/k1_ab.py --config C3 --n0 8000000 --reps 3 - > gpurun_out/r3b_${lib}_C3_8M.log 2>&1
  KNNG_LIB=$L/$lib.so timeout 900 python scripts/k1_ab.py --config C4 --n0 500000 --reps 3 - > gpurun_out/r3b_${lib}_C4.log 2>&1
done
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/r3b_bench.json 2> gpurun_out/r3b_bench.err; echo "bench rc=$?" >> gpurun_out/r3b_bench.err
