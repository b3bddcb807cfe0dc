#!/bin/bash
# A/B timing of library variants on the same box: tools/ab.sh libA.so libB.so ...
for rep in 1 2; do
for lib in "$@"; do
  for grid in 2x4 1x1; do
    PTYCHO_LIB=$lib timeout 900 python bench.py --grid $grid --steps 1 --warmup 1 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$grid', round(d['value'],1), 'ms/probe', round(d['ms_per_step']/4158,3), 'bwd_us', round(d['roofline']['isolated']['ms_per_launch']*1e3,2), 'frac', round(d['roofline']['frac'],3))"
  done
done
done
