# bulk-copy gathers on the two-stage plan (one barrier per stage): forced-path parity, then the C1 A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "bulk or long_walks or smem" > gpurun_out/r3p_par.log 2>&1; echo "rc=$?" >> gpurun_out/r3p_par.log
if grep -q "rc=0" gpurun_out/r3p_par.log; then
  timeout 600 python scripts/k1_ab.py --config C1 --n0 100000 --reps 5 KNNG_BULK2=0 KNNG_BULK2=1 KNNG_BULK2=0 KNNG_BULK2=1 > gpurun_out/r3p_C1.log 2>&1
  timeout 600 python scripts/k1_ab.py --config C2 --n0 1000000 --reps 3 - > gpurun_out/r3p_C2.log 2>&1
fi
