mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 --durations=15 > gpurun_out/r2e_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_pytest.log
timeout 1500 python scripts/sweeps.py --configs C1,C2,C4 --n0 100000 > gpurun_out/r2e_sweeps.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_sweeps.log
