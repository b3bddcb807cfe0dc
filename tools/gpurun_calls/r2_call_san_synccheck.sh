timeout 600 python tools/sanitize_tiny.py > gpurun_out/san_plain_synccheck.log 2>&1 && \
timeout 1500 compute-sanitizer --tool synccheck  --print-limit 50 python tools/sanitize_tiny.py > gpurun_out/san_synccheck.log 2>&1; echo rc=$?; tail -5 gpurun_out/san_synccheck.log
