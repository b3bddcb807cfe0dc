python bench.py --config lt_large --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/r2_bench_lt_large.json 2> gpurun_out/r2_bench_lt_large.err; cut -c1-250 gpurun_out/r2_bench_lt_large.json; tail -c 300 gpurun_out/r2_bench_lt_large.err
python bench.py --stash-free --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_stash_free.json 2>/dev/null; cut -c1-250 gpurun_out/r2_bench_stash_free.json
python bench.py --halo 60 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_halo60.json 2>/dev/null; cut -c1-250 gpurun_out/r2_bench_halo60.json
