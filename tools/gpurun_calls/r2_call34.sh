# final bench lines after the e2e warm-up / async change: N=4, N=2, N=1
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 > gpurun_out/r2_final3_n4.json 2> gpurun_out/r2_final3_n4.err
grep '^{' gpurun_out/r2_final3_n4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=4', d['value'], d['e2e'])"
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 2 > gpurun_out/r2_final3_n2.json 2> gpurun_out/r2_final3_n2.err
grep '^{' gpurun_out/r2_final3_n2.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=2', d['value'], d['e2e'])"
timeout 1200 python bench.py > gpurun_out/r2_final3_n1.json 2> gpurun_out/r2_final3_n1.err
grep '^{' gpurun_out/r2_final3_n1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=1', d['value'], d['e2e'], d['clocks'])"
