#!/bin/bash
# engine geometry x gradient form x config
for cfg in pythia rho llama; do
  for eng in 0 1; do
    for grad in scaled unscaled; do
      timeout 200 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux --gradient $grad --engine $eng 2>&1 | tail -1 | python -c "
import json,sys
l=sys.stdin.read()
try:
  d=json.loads(l); print('$cfg engine $eng $grad', '| loss_ms %.3f | eff %.0f GB/s frac %.3f | status %s' % (d['roofline']['loss_ms_mean'], d['roofline']['achieved'], d['roofline']['frac'], d['status']))
except Exception as e: print('$cfg $eng $grad FAILED', l[-300:])
"
    done
  done
done
