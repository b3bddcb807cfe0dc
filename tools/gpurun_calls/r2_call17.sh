bash tools/ab.sh build/libptycho_vote1.so build/libptycho_tma3.so > gpurun_out/r2_ab_vote1.txt 2>&1; cat gpurun_out/r2_ab_vote1.txt
bash tools/gpurun_calls/r2_call_hve.sh
