export PTYCHO_DEBUG_SYNC=1 PTYCHO_NO_GRAPH=1
for args in "1024 4 1536 12 81" "64 4 128 16 17" "256 4 512 9 57"; do PTYCHO_LIB=build/libptycho_dist.so timeout 120 python tools/diag_tma3.py $args; done
unset PTYCHO_DEBUG_SYNC PTYCHO_NO_GRAPH
bash tools/ab.sh build/libptycho_dist.so build/libptycho_u8.so > gpurun_out/r2_ab_dist.txt 2>&1; cat gpurun_out/r2_ab_dist.txt
for lib in build/libptycho_dist.so build/libptycho_u8.so; do for cfg in small appp; do
PTYCHO_LIB=$lib timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$cfg', round(d['value'],1))"
done; done
