python tools/prof_chain.py --grid 2x4 --probes 2 > gpurun_out/prof_plain_final.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pass_kernel --csv --log-file gpurun_out/r2_launches_chain.csv python tools/prof_chain.py --grid 2x4 --probes 2 > gpurun_out/r2_ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pass_kernel -s 150 -c 1 -o gpurun_out/r2_final_bwd python tools/prof_chain.py --grid 2x4 --probes 1 > gpurun_out/r2_ncu_final.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pass_kernel -s 50 -c 1 -o gpurun_out/r2_final_fwd python tools/prof_chain.py --grid 2x4 --probes 1 >> gpurun_out/r2_ncu_final.log 2>&1
tail -3 gpurun_out/r2_ncu_final.log; wc -l gpurun_out/r2_launches_chain.csv
