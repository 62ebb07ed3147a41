mkdir -p gpurun_out; timeout 300 ./scripts/micro/eval_micro > gpurun_out/micro.log 2>&1
