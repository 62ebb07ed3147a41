# sets: lane-slot size A/B on C4 (2M sets, P = 8, one 4096 batch), with parity of the small-slot path first
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "set-slots or bulk" > gpurun_out/r3k_par.log 2>&1; echo "rc=$?" >> gpurun_out/r3k_par.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "jaccard" > gpurun_out/r3k_par2.log 2>&1; echo "rc=$?" >> gpurun_out/r3k_par2.log
timeout 1500 python scripts/k1_ab.py --config C4 --n0 2000000 --reps 3 KNNG_SET_SLOTCH=16 KNNG_SET_SLOTCH=12 KNNG_SET_SLOTCH=10 KNNG_SET_SLOTCH=8 KNNG_SET_SLOTCH=16 KNNG_SET_SLOTCH=12 > gpurun_out/r3k_C4.log 2>&1
