#!/bin/bash
# unscaled: exp2 split x lookahead sweep (geometry 0)
CFG=${1:-pythia}
for args in "--exp2-split 0" "--exp2-split 1" "--exp2-split 2" "--exp2-split 5" "--exp2-split 6" "--lookahead 0" "--lookahead 2" "--ctas-per-sm 3"; do
  timeout 120 python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux --gradient unscaled $args 2>&1 | tail -1 | python -c "
import json,sys
l=sys.stdin.read()
try:
  d=json.loads(l); print('$CFG $args', '| loss_ms %.3f | eff %.0f GB/s frac %.3f | status %s | clk %s' % (d['roofline']['loss_ms_mean'], d['roofline']['achieved'], d['roofline']['frac'], d['status'], d['clocks']['sm_mhz']))
except Exception as e: print('$args FAILED', l[-300:])
"
done
