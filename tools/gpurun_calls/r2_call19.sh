bash tools/ab.sh build/libptycho_u8.so build/libptycho_vote1.so build/libptycho_s8.so > gpurun_out/r2_ab_unroll.txt 2>&1; cat gpurun_out/r2_ab_unroll.txt
python tools/prof_chain.py --grid 1x1 --probes 1 > gpurun_out/prof_plain19.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pass_kernel -s 150 -c 1 -o gpurun_out/r2_bwd_lone_vote1 python tools/prof_chain.py --grid 1x1 --probes 1 > gpurun_out/r2_ncu19.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pass_kernel -s 50 -c 1 -o gpurun_out/r2_fwd_lone_vote1 python tools/prof_chain.py --grid 1x1 --probes 1 >> gpurun_out/r2_ncu19.log 2>&1
tail -2 gpurun_out/r2_ncu19.log
