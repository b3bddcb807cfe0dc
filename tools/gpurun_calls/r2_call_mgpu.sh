nvidia-smi -L > gpurun_out/r2_mgpu_smi.txt
timeout 1500 python -m pytest tests/test_multigpu.py -x -q -s > gpurun_out/r2_mgpu_tests.log 2>&1; tail -3 gpurun_out/r2_mgpu_tests.log
for n in 2 4; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $n --steps 3 --warmup 3 > gpurun_out/r2_bench_n$n.json 2> gpurun_out/r2_bench_n$n.err
  cut -c1-300 gpurun_out/r2_bench_n$n.json; tail -c 300 gpurun_out/r2_bench_n$n.err
done
