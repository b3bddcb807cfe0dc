export PTYCHO_DEBUG_SYNC=1 PTYCHO_NO_GRAPH=1
for args in "1024 4 1536 12 81" "64 4 128 16 17" "256 4 512 9 57"; do PTYCHO_LIB=build/libptycho_sbulk.so timeout 120 python tools/diag_tma3.py $args; done
unset PTYCHO_DEBUG_SYNC PTYCHO_NO_GRAPH
PTYCHO_LIB=build/libptycho_sbulk_dbg.so timeout 900 python tools/ordering_run.py > gpurun_out/sbulk_dbg.jsonl 2>&1; cut -c1-200 gpurun_out/sbulk_dbg.jsonl
PTYCHO_LIB=build/libptycho_sbulk.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_stash_free.py -x -q 2>&1 | tail -2
bash tools/ab.sh build/libptycho_sbulk.so build/libptycho_red.so > gpurun_out/r2_ab_sbulk.txt 2>&1; cat gpurun_out/r2_ab_sbulk.txt
