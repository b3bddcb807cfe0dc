GRIDS="2x4" bash tools/ab.sh build/libptycho_fwd4.so build/libptycho_final.so > gpurun_out/r2_ab_fwd4.txt 2>&1; cat gpurun_out/r2_ab_fwd4.txt
