export PTYCHO_DEBUG_SYNC=1 PTYCHO_NO_GRAPH=1
for args in "1024 4 1536 12 81" "1024 4 1536 743 477"; do PTYCHO_LIB=build/libptycho_bwd3.so PTYCHO_HIGH_OCC=1 timeout 120 python tools/diag_tma3.py $args; done
unset PTYCHO_DEBUG_SYNC PTYCHO_NO_GRAPH
PTYCHO_LIB=build/libptycho_bwd3.so python -m pytest tests/test_gpu_fullsize.py -k "lt_small-5" -x -q -s 2>&1 | grep -E "grad|passed|failed"
PTYCHO_LIB=build/libptycho_bwd3.so python -m pytest tests/test_gpu_recon_large.py -k "lt_geometry" -x -q -s 2>&1 | grep -E "rel|passed|failed"
bash tools/ab.sh build/libptycho_bwd3.so build/libptycho_red.so > gpurun_out/r2_ab_bwd3.txt 2>&1; cat gpurun_out/r2_ab_bwd3.txt
