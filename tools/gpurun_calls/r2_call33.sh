# e2e async-upload A/B after the e2e warm-up fix (interleaved, N=1 and N=2)
for rep in 1 2; do
for a in on off; do
timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 3 --e2e-async $a 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=1', '$a', round(d['value'],1), round(d['e2e']['value'],1), round(d['e2e']['ms_per_step'],1))" | tee -a gpurun_out/e2e_async_ab2.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 1 --warmup 3 --e2e-steps 3 --e2e-async $a 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=2', '$a', round(d['value'],1), round(d['e2e']['value'],1), round(d['e2e']['ms_per_step'],1))" | tee -a gpurun_out/e2e_async_ab2.txt
done
done
