# copy-stream timeline of the async load while the chains run (PTYCHO_AMP_TRACE)
PTYCHO_AMP_TRACE=1 timeout 900 python tools/e2e_overlap.py 2>&1 | grep '^{\|AMP_TRACE' | tee -a gpurun_out/e2e_overlap6.jsonl
