# host time of the async load call (does it block?), chunk 8 and 520
for c in 8 520; do PTYCHO_AMP_CHUNK=$c timeout 900 python tools/e2e_overlap.py 2>&1 | grep '^{' | tee -a gpurun_out/e2e_overlap4.jsonl; done
