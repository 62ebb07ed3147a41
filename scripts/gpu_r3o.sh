# final confirmation of the committed tree: smoke, the full GPU suite, the default bench line (C3)
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f6_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f6_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f6_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f6_pytest.log
timeout 1200 python bench.py > gpurun_out/f6_bench.json 2> gpurun_out/f6_bench.err; echo "bench rc=$?" >> gpurun_out/f6_bench.err
