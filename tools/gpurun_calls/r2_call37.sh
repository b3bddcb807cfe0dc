# overlapped-upload interference with the chains at N=1 (chunk 8 default, 64, 1)
for c in 8 64 1; do PTYCHO_AMP_CHUNK=$c timeout 900 python tools/e2e_overlap.py 2>&1 | grep '^{' | tee -a gpurun_out/e2e_overlap.jsonl; done
