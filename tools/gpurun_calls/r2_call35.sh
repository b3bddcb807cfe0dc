# lone chain (1x1 grid: the per-GPU case at N=8) -- launch list + ncu --set full of BWD_MID and FWD_MID
python tools/prof_chain.py --grid 1x1 --probes 2 > gpurun_out/prof_lone.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pass_kernel --csv --log-file gpurun_out/r2_launches_lone.csv python tools/prof_chain.py --grid 1x1 --probes 2 > gpurun_out/r2_ncu_lone_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pass_kernel -s 150 -c 1 -o gpurun_out/r2_lone_bwd python tools/prof_chain.py --grid 1x1 --probes 1 > gpurun_out/r2_ncu_lone.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pass_kernel -s 50 -c 1 -o gpurun_out/r2_lone_fwd python tools/prof_chain.py --grid 1x1 --probes 1 >> gpurun_out/r2_ncu_lone.log 2>&1
tail -3 gpurun_out/r2_ncu_lone.log; wc -l gpurun_out/r2_launches_lone.csv
