# confirmation of the committed tree: smoke, the GPU tests, the default bench line (C3).
mkdir -p gpurun_out
nvidia-smi > gpurun_out/c_nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/c_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/c_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/c_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c_pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/c_bench.json 2> gpurun_out/c_bench.err; echo "bench rc=$?" >> gpurun_out/c_bench.err
