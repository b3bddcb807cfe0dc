#!/bin/bash
# A/B timing of environment variants on the same box: tools/ab_env.sh "PTYCHO_PERSIST=0" "PTYCHO_PERSIST=1" ...
for rep in 1 2; do
for envs in "$@"; do
  for grid in 2x4 1x1; do
    env $envs timeout 900 python bench.py --grid $grid --steps 1 --warmup 1 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$envs', '$grid', round(d['value'],1), 'ms/probe', round(d['ms_per_step']/4158,3), 'loss', d['loss_after'])"
  done
done
done
