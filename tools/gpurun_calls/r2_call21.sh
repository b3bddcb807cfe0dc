export PTYCHO_LIB=build/libptycho_cl.so
timeout 600 python tools/ordering_run.py tiny_2x2 tiny_hve small_1x1 small_2x2 > gpurun_out/cl_on.jsonl 2> gpurun_out/cl_on.err; tail -3 gpurun_out/cl_on.err
PTYCHO_CLUSTER=0 timeout 600 python tools/ordering_run.py tiny_2x2 tiny_hve small_1x1 small_2x2 > gpurun_out/cl_off.jsonl 2> gpurun_out/cl_off.err
python - <<'PY'
import json
a=[json.loads(l) for l in open('gpurun_out/cl_on.jsonl')]; b=[json.loads(l) for l in open('gpurun_out/cl_off.jsonl')]
for x,y in zip(a,b): print(x['case'], 'cluster==standalone', x['sha']==y['sha'], x['losses'], y['losses'])
PY
for cl in 1 0; do for cfg in small appp; do
PTYCHO_CLUSTER=$cl timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu --no-e2e 2>gpurun_out/cl_bench_$cfg$cl.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cluster=$cl', '$cfg', round(d['value'],1), round(d['ms_per_step'],2), 'ms/iter')"
done; done
