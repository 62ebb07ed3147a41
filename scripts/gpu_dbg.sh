mkdir -p gpurun_out
timeout 120 python -m pytest tests/test_gpu_fullsize.py -x -q -k "long_walk" > gpurun_out/dbg1.log 2>&1; echo "rc=$?" >> gpurun_out/dbg1.log
timeout 120 python -m pytest tests/test_gpu_parity.py -x -q -k "w3 or search_matches" > gpurun_out/dbg2.log 2>&1; echo "rc=$?" >> gpurun_out/dbg2.log
