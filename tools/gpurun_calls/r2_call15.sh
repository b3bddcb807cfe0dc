bash tools/ab.sh build/libptycho_tma3.so build/libptycho_tma2.so build/libptycho_notma3.so > gpurun_out/r2_ab_tma3.txt 2>&1; cat gpurun_out/r2_ab_tma3.txt
