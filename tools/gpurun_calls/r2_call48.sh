# async measurement upload by kernels through the pinned buffer's device alias vs copy-engine copies
timeout 600 python -m pytest tests -m gpu -x -q -k "async or measurement" > gpurun_out/r2_up_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/r2_up_tests.log
timeout 900 python tools/e2e_overlap.py 2>&1 | grep '^{' | sed 's/^{/{"mode": "kernel8", /' | tee -a gpurun_out/e2e_overlap10.jsonl
PTYCHO_AMP_UPLOAD_CTAS=16 timeout 900 python tools/e2e_overlap.py 2>&1 | grep '^{' | sed 's/^{/{"mode": "kernel16", /' | tee -a gpurun_out/e2e_overlap10.jsonl
PTYCHO_AMP_CE=1 timeout 900 python tools/e2e_overlap.py 2>&1 | grep '^{' | sed 's/^{/{"mode": "ce", /' | tee -a gpurun_out/e2e_overlap10.jsonl
