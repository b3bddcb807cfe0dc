python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python -m pytest tests -m gpu -x -q > gpurun_out/r2_head_tests.log 2>&1; tail -2 gpurun_out/r2_head_tests.log
python bench.py > gpurun_out/r2_head_bench.json 2> gpurun_out/r2_head_bench.err; cut -c1-300 gpurun_out/r2_head_bench.json
