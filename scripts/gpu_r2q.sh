mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x --timeout 600 -k "forced" > gpurun_out/r2q_pytest0.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_pytest0.log
KNNG_NS2G=1 timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x --timeout 600 -k "forced or partitioned or insert_C" > gpurun_out/r2q_pytest1.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_pytest1.log
timeout 600 python scripts/k1_ab.py --config C3 --n0 2000000 --reps 3 - KNNG_NS2G=1 > gpurun_out/r2q_C3.log 2>&1
timeout 600 python scripts/k1_ab.py --config C2 --n0 1000000 --reps 3 - KNNG_NS2G=1 > gpurun_out/r2q_C2.log 2>&1
