# raw DMA in 32 MiB chunks + events concurrent with an iteration
timeout 900 python tools/e2e_overlap.py 2>&1 | grep '^{' | tee -a gpurun_out/e2e_overlap5.jsonl
