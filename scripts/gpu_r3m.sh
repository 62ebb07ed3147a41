# final confirmation after the B = 1 shared-memory rows: smoke, the full GPU suite, the C0 line
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f5_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f5_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f5_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f5_pytest.log
timeout 300 python scripts/prof_c0.py > gpurun_out/f5_c0_srows.log 2>&1
timeout 600 python bench.py --config C0 --steps 20 --warmup 3 > gpurun_out/f5_bench_C0.json 2> gpurun_out/f5_bench_C0.err
