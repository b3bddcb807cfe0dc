# host-side chunk gate instead of cross-stream event waits: overlap timing, async parity tests, bench N=1
timeout 900 python tools/e2e_overlap.py 2>&1 | grep '^{' | tee -a gpurun_out/e2e_overlap9.jsonl
timeout 900 python -m pytest tests -m gpu -x -q -k "async or measurement or stitch or profile" > gpurun_out/r2_gate_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r2_gate_tests.log
timeout 1200 python bench.py --no-cpu > gpurun_out/r2_gate_bench.json 2> gpurun_out/r2_gate_bench.err
grep '^{' gpurun_out/r2_gate_bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=1', d['value'], d['e2e'], d['clocks'])"
