python -m pytest tests -m gpu -x -q -s > gpurun_out/r2_gputests18.log 2>&1; tail -3 gpurun_out/r2_gputests18.log
python bench.py --steps 3 --warmup 3 > gpurun_out/r2_bench18.json 2> gpurun_out/r2_bench18.err; tail -c 600 gpurun_out/r2_bench18.err; cut -c1-400 gpurun_out/r2_bench18.json
