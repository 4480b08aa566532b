#!/bin/bash
# unscaled-gradient sweep: engine geometry builds x row_gap
CFG=${1:-pythia}
for lib in default build_variants/libodpo_*.so; do
  for gap in 0 1; do
    if [ "$lib" = default ]; then L=""; else L="ODPO_LIB=$PWD/$lib"; fi
    env $L timeout 120 python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux --gradient unscaled --row-gap $gap 2>&1 | tail -1 | python -c "
import json,sys
l=sys.stdin.read()
try:
  d=json.loads(l); print('$(basename $lib) gap $gap', '| loss_ms %.3f | eff %.0f GB/s frac %.3f | ref_ms %.3f (%.0f GB/s) | status %s' % (d['roofline']['loss_ms_mean'], d['roofline']['achieved'], d['roofline']['frac'], d['ref_pass_ms'], d['ref_pass_gbs'], d['status']))
except Exception as e: print('$(basename $lib) gap $gap FAILED', l[-300:])
"
  done
done
