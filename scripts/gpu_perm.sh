# permutation draws + perm_e: parity suite, A/B of perm_e (identical results required), the default line
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/p_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/p_pytest_gpu.log
S="- KNNG_PERM_E=0 -"
timeout 900 python scripts/k1_ab.py --config C3 --n0 8000000 --reps 3 $S > gpurun_out/p_ab_C3_8M.txt 2>&1
timeout 400 python scripts/k1_ab.py --config C2 --n0 1000000 --reps 3 $S > gpurun_out/p_ab_C2.txt 2>&1
timeout 400 python scripts/k1_ab.py --config C4 --n0 500000 --reps 3 $S > gpurun_out/p_ab_C4_500k.txt 2>&1
timeout 1200 python bench.py > gpurun_out/p_bench.json 2> gpurun_out/p_bench.err
