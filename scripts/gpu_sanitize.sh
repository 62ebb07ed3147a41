mkdir -p gpurun_out
timeout 600 python scripts/sanitize_case.py > gpurun_out/san_plain.log 2>&1 && \
timeout 1800 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_case.py > gpurun_out/san_memcheck.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/san_memcheck.log
