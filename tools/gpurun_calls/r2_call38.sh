# unrelated 17 GB H2D DMA concurrent with an iteration: does raw DMA slow the chains?
timeout 900 python tools/e2e_overlap.py 2>&1 | grep '^{' | tee -a gpurun_out/e2e_overlap2.jsonl
