GRIDS="1x1" bash tools/ab_env.sh "PTYCHO_HIGH_OCC=0" "PTYCHO_HIGH_OCC=1" > gpurun_out/r2_ab_lone_occ.txt 2>&1; cat gpurun_out/r2_ab_lone_occ.txt
