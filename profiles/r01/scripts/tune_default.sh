#!/bin/bash
for lib in default build_variants/libodpo_C2.so build_variants/libodpo_C4.so build_variants/libodpo_C8.so; do
  for args in "--lookahead 1" "--lookahead 0" "--schedule two_pass"; do
    if [ "$lib" = default ]; then L=""; else L="ODPO_LIB=$PWD/$lib"; fi
    env $L timeout 60 python bench.py --config ${CFG:-pythia} --steps 10 --warmup 3 --no-cpu --no-e2e $args 2>&1 | tail -1 | python -c "
import json,sys
l=sys.stdin.read()
try:
  d=json.loads(l); print('$(basename $lib) $args', '| pairs/s %.0f | loss_ms %.3f | eff %.0f GB/s | ref_ms %.3f (%.0f GB/s) | status %s' % (d['value'], d['roofline']['loss_ms_mean'], d['roofline']['achieved'], d['ref_pass_ms'], d['ref_pass_gbs'], d['status']))
except Exception as e: print('$(basename $lib) $args FAILED', l[-300:])
"
  done
done
