mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x --timeout 600 -k "forced or long_walk" > gpurun_out/r2r_pytest0.log 2>&1; echo "rc=$?" >> gpurun_out/r2r_pytest0.log
timeout 600 python scripts/k1_ab.py --config C3 --n0 2000000 --reps 3 - KNNG_WKC=0 > gpurun_out/r2r_C3.log 2>&1
timeout 600 python scripts/k1_ab.py --config C2 --n0 1000000 --reps 3 - KNNG_WKC=0 > gpurun_out/r2r_C2.log 2>&1
timeout 300 python scripts/k1_ab.py --config C1 --n0 100000 --reps 3 - KNNG_WKC=0 > gpurun_out/r2r_C1.log 2>&1
