# diagnostic: chains not waiting for the chunk events (racy; timing only)
PTYCHO_AMP_TRACE=1 PTYCHO_AMP_NOWAIT_DIAG=1 timeout 900 python tools/e2e_overlap.py 2>&1 | grep '^{\|AMP_TRACE' | tee -a gpurun_out/e2e_overlap7.jsonl
