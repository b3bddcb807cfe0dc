timeout 1500 python tools/hve_compare.py seam > gpurun_out/r2_hve_seam.jsonl 2> gpurun_out/r2_hve_seam.err; tail -3 gpurun_out/r2_hve_seam.err
timeout 1500 python tools/hve_compare.py perf > gpurun_out/r2_hve_perf.jsonl 2> gpurun_out/r2_hve_perf.err; tail -3 gpurun_out/r2_hve_perf.err
cat gpurun_out/r2_hve_seam.jsonl; cut -c1-600 gpurun_out/r2_hve_perf.jsonl
