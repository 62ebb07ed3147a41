mkdir -p gpurun_out
L=$PWD/paper_1602_06819_b200
for lib in libknng libknng_mb7 libknng_mb8; do
  KNNG_LIB=$L/$lib.so timeout 600 python scripts/k1_ab.py --config C3 --n0 2000000 --reps 3 - > gpurun_out/r2n_${lib}_C3.log 2>&1
done
KNNG_LIB=$L/libknng_prof.so KNNG_PROFILE=1 timeout 300 python scripts/k1_ab.py --config C3 --n0 2000000 --reps 1 - > gpurun_out/r2n_prof_C3.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r2n_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2n_pytest.log
