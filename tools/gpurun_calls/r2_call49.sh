# final validation with upload kernels: GPU suite (4 GPUs), bench N=4 / N=2 / N=1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/final5_gpu_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/final5_gpu_tests.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus 4 > gpurun_out/r2_final5_n4.json 2> gpurun_out/r2_final5_n4.err
grep '^{' gpurun_out/r2_final5_n4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=4', d['value'], d['e2e']['value'])"
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29552 bench.py --gpus 2 > gpurun_out/r2_final5_n2.json 2> gpurun_out/r2_final5_n2.err
grep '^{' gpurun_out/r2_final5_n2.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=2', d['value'], d['e2e']['value'])"
timeout 1200 python bench.py > gpurun_out/r2_final5_n1.json 2> gpurun_out/r2_final5_n1.err
grep '^{' gpurun_out/r2_final5_n1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=1', d['value'], d['e2e']['value'], d['clocks'])"
