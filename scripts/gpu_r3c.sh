# string measures: GPU parity tests first, then the whole GPU suite
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_strings.py -x -q > gpurun_out/r3c_strings.log 2>&1; echo "rc=$?" >> gpurun_out/r3c_strings.log
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_strings.py > gpurun_out/r3c_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r3c_pytest.log
