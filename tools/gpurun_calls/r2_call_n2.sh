timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 2 --warmup 3 --no-e2e > gpurun_out/r2_bench3_n2.json 2> gpurun_out/r2_bench3_n2.err
grep '^{' gpurun_out/r2_bench3_n2.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['appp'], d['breakdown'])"
