export PTYCHO_DEBUG_SYNC=1 PTYCHO_NO_GRAPH=1
for args in "1024 4 1536 12 81" "1024 4 1536 743 477" "1024 4 1536 768 768" "64 4 128 16 17" "256 4 512 9 57"; do
  timeout 120 python tools/diag_tma3.py $args
done
unset PTYCHO_DEBUG_SYNC PTYCHO_NO_GRAPH
python -m pytest tests/test_gpu_parity.py tests/test_gpu_hve.py tests/test_gpu_stash_free.py -x -q > gpurun_out/r2_tma2_tests.log 2>&1; tail -2 gpurun_out/r2_tma2_tests.log
python -m pytest tests/test_gpu_fullsize.py -k "lt_small-5 or appp" -x -q -s 2>&1 | grep -E "grad|passed|failed"
bash tools/ab.sh build/libptycho_tma2.so build/libptycho_notma2.so build/libptycho_f2.so > gpurun_out/r2_ab_tma2.txt 2>&1; cat gpurun_out/r2_ab_tma2.txt
