for env in "PTYCHO_PERSIST=0" "PTYCHO_PERSIST=1"; do for cfg in small appp; do
env $env timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$env', '$cfg', round(d['value'],1))"
done; done
