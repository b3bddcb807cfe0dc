timeout 600 python tools/sanitize_tiny.py > gpurun_out/san_plain_memcheck.log 2>&1 && \
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 50 python tools/sanitize_tiny.py > gpurun_out/san_memcheck.log 2>&1; echo rc=$?; tail -5 gpurun_out/san_memcheck.log
