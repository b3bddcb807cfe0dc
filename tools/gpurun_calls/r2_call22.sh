export PTYCHO_DEBUG_SYNC=1 PTYCHO_NO_GRAPH=1
for args in "1024 4 1536 12 81" "64 4 128 16 17" "256 4 512 9 57"; do PTYCHO_LIB=build/libptycho_red.so timeout 120 python tools/diag_tma3.py $args; done
unset PTYCHO_DEBUG_SYNC PTYCHO_NO_GRAPH
PTYCHO_LIB=build/libptycho_red.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_hve.py -x -q 2>&1 | tail -2
PTYCHO_LIB=build/libptycho_red.so python -m pytest tests/test_gpu_fullsize.py -k "lt_small-5 or appp" -x -q -s 2>&1 | grep -E "grad|passed|failed"
bash tools/ab.sh build/libptycho_red.so build/libptycho_dist.so > gpurun_out/r2_ab_red.txt 2>&1; cat gpurun_out/r2_ab_red.txt
