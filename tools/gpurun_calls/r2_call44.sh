# chunk waits skipped when the chunk has already landed (cudaEventQuery)
PTYCHO_AMP_TRACE=1 timeout 900 python tools/e2e_overlap.py 2>&1 | grep '^{\|AMP_TRACE' | tee -a gpurun_out/e2e_overlap8.jsonl
timeout 900 python tools/e2e_overlap.py 2>&1 | grep '^{' | tee -a gpurun_out/e2e_overlap8.jsonl
