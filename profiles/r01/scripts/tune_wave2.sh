#!/bin/bash
for args in "--schedule wave --row-gap 0 --engine 1" "--schedule wave --row-gap 1 --engine 1" "--schedule fused --engine 1" "--schedule wave --row-gap 1 --lookahead 2" "--schedule wave --row-gap 1 --lookahead 3"; do
    ODPO_LIB=$PWD/build_variants/libodpo_WB90.so timeout 120 python bench.py --config pythia --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux $args 2>&1 | tail -1 | python -c "
import json,sys
l=sys.stdin.read()
try:
  d=json.loads(l); print('WB90 $args', '| pairs/s %.0f | loss_ms %.3f | eff %.0f GB/s frac %.3f | status %s' % (d['value'], d['roofline']['loss_ms_mean'], d['roofline']['achieved'], d['roofline']['frac'], d['status']))
except Exception as e: print('$args FAILED', l[-300:])
"
done
