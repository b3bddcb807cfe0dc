# e2e leg breakdown at N=2 and N=4 (raw pinned H2D, staged/async load, stitch, iterate)
for N in 4 2; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N tools/e2e_parts.py > gpurun_out/e2e_parts_n$N.jsonl 2> gpurun_out/e2e_parts_n$N.err
tail -3 gpurun_out/e2e_parts_n$N.jsonl; tail -3 gpurun_out/e2e_parts_n$N.err
done
timeout 600 python tools/e2e_parts.py > gpurun_out/e2e_parts_n1.jsonl 2> gpurun_out/e2e_parts_n1.err; tail -2 gpurun_out/e2e_parts_n1.jsonl
