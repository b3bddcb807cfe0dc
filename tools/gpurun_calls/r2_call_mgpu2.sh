timeout 1500 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/r2_mgpu2_tests.log 2>&1; tail -2 gpurun_out/r2_mgpu2_tests.log
for n in 2 4; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $n --steps 3 --warmup 3 > gpurun_out/r2_bench2_n$n.json 2> gpurun_out/r2_bench2_n$n.err
  grep '^{' gpurun_out/r2_bench2_n$n.json | cut -c1-250
done
python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench2_n1.json 2> gpurun_out/r2_bench2_n1.err; cut -c1-250 gpurun_out/r2_bench2_n1.json
