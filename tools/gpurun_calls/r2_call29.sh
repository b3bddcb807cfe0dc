for it in 100 300; do timeout 1200 python tools/hve_compare.py seam $it > gpurun_out/r2_hve_seam_$it.jsonl 2>/dev/null; cat gpurun_out/r2_hve_seam_$it.jsonl; done
