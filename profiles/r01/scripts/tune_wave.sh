#!/bin/bash
for lib in default build_variants/libodpo_WB50.so build_variants/libodpo_WB90.so; do
  if [ "$lib" = default ]; then L=""; else L="ODPO_LIB=$PWD/$lib"; fi
  for args in "--schedule fused" "--schedule wave --row-gap 0" "--schedule wave --row-gap 1"; do
    env $L timeout 120 python bench.py --config pythia --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux $args 2>&1 | tail -1 | python -c "
import json,sys
l=sys.stdin.read()
try:
  d=json.loads(l); print('$(basename $lib) $args', '| pairs/s %.0f | loss_ms %.3f | eff %.0f GB/s frac %.3f | status %s' % (d['value'], d['roofline']['loss_ms_mean'], d['roofline']['achieved'], d['roofline']['frac'], d['status']))
except Exception as e: print('$(basename $lib) $args FAILED', l[-300:])
"
  done
done
