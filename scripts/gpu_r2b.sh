# new K1: fast GPU tests first, then quick bench lines (each command under its own timeout)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -rf --timeout 300 -k "not full_prefix and not C0_full" > gpurun_out/r2b_pytest.log 2>&1; rc=$?; echo "pytest rc=$rc" >> gpurun_out/r2b_pytest.log
if [ $rc -ne 0 ]; then exit 0; fi
KNNG_PROFILE=1 timeout 400 python bench.py --config C3 --n0 2000000 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_C3_2M.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_C3_2M.log
KNNG_PROFILE=1 timeout 300 python bench.py --config C1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_C1.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_C1.log
KNNG_PROFILE=1 timeout 300 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_C2.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_C2.log
KNNG_PROFILE=1 timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_C3.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_C3.log
