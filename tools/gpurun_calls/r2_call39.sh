# hardware work-queue sharing: CUDA_DEVICE_MAX_CONNECTIONS 8 (default) vs 32
for rep in 1 2; do
for c in 32 8; do CUDA_DEVICE_MAX_CONNECTIONS=$c timeout 900 python tools/e2e_overlap.py 2>&1 | grep '^{' | sed "s/^{/{\"conn\": $c, /" | tee -a gpurun_out/e2e_overlap3.jsonl; done
done
