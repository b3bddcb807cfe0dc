#!/bin/bash
# A/B of environment settings on the same box: GRIDS="2x4 1x1" tools/ab_env.sh "VAR=a" "VAR=b" ...
for rep in 1 2; do
for envs in "$@"; do
  for grid in ${GRIDS:-2x4}; do
    env $envs timeout 900 python bench.py --grid $grid --steps 1 --warmup 1 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$envs', '$grid', round(d['value'],1), 'frac', round(d['roofline']['frac'],3))"
  done
done
done
