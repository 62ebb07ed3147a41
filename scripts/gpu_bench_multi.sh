# N=1 bench + a 2-rank plumbing run of the multi-GPU bench path on ONE GPU (gloo, host-staged exchange:
# no kernel waits on another rank).  Not a performance number.
mkdir -p gpurun_out
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n1.log
KNNG_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_n2_plumbing.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n2_plumbing.log
