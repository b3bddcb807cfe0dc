python -m pytest tests -m gpu -x -q -s > gpurun_out/r2_final_tests.log 2>&1; tail -3 gpurun_out/r2_final_tests.log
python bench.py --steps 5 --warmup 3 > gpurun_out/r2_final_bench.json 2> gpurun_out/r2_final_bench.err; cut -c1-300 gpurun_out/r2_final_bench.json; tail -c 300 gpurun_out/r2_final_bench.err
python bench.py --grid 1x1 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_final_bench_1x1.json 2>/dev/null; cut -c1-200 gpurun_out/r2_final_bench_1x1.json
for cfg in small appp; do python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_final_bench_$cfg.json 2>/dev/null; cut -c1-200 gpurun_out/r2_final_bench_$cfg.json; done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_final_ref.json 2> gpurun_out/r2_final_ref.err; cut -c1-400 gpurun_out/r2_final_ref.json
