# session-3 baseline check of the restored tree: smoke, GPU tests, default bench line (C3)
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r3a_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r3a_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r3a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r3a_pytest.log
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/r3a_bench.json 2> gpurun_out/r3a_bench.err; echo "bench rc=$?" >> gpurun_out/r3a_bench.err
