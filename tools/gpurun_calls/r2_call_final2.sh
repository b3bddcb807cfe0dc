python -m pytest tests -m gpu -x -q > gpurun_out/r2_final2_tests.log 2>&1; tail -2 gpurun_out/r2_final2_tests.log
python bench.py --steps 5 --warmup 3 > gpurun_out/r2_final2_bench.json 2> gpurun_out/r2_final2_bench.err; cut -c1-200 gpurun_out/r2_final2_bench.json
python bench.py --steps 3 --warmup 3 --no-cpu --e2e-async on --e2e-steps 3 > gpurun_out/r2_final2_bench_async.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/r2_final2_bench_async.json')); print('async e2e', d['value'], d['e2e'])"
python bench.py --grid 1x1 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_final2_bench_1x1.json 2>/dev/null; cut -c1-200 gpurun_out/r2_final2_bench_1x1.json
