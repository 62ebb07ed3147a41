# round-2 check: GPU tests (with durations) and the default bench line (C3 at G=1)
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu > gpurun_out/lscpu.txt 2>&1; free -g > gpurun_out/free.txt
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 1500 --durations=25 > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2a_pytest.log
timeout 1500 python bench.py > gpurun_out/r2a_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r2a_bench.log
