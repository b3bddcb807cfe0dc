python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
GRIDS="2x4" bash tools/ab_env.sh "PTYCHO_TILE_STREAMS=4" "PTYCHO_TILE_STREAMS=3" "PTYCHO_TILE_STREAMS=6" "PTYCHO_TILE_STREAMS=8" "PTYCHO_HIGH_OCC=0" > gpurun_out/r2_ab_env.txt 2>&1; cat gpurun_out/r2_ab_env.txt
