mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "fast_path or C0 or edge" > gpurun_out/r2i_pytest0.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_pytest0.log
timeout 300 python bench.py --config C0 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/r2i_bench_C0.json 2> gpurun_out/r2i_bench_C0.err
KNNG_NO_KT=1 timeout 300 python bench.py --config C0 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/r2i_bench_C0_nokt.json 2> gpurun_out/r2i_bench_C0_nokt.err
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/r2i_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_pytest.log
