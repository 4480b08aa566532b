#!/bin/bash
for lib in default build_variants/libodpo_BR.so; do
  if [ "$lib" = default ]; then L=""; else L="ODPO_LIB=$PWD/$lib"; fi
  for cfg in pythia rho llama; do
    env $L timeout 200 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux 2>&1 | tail -1 | python -c "
import json,sys
l=sys.stdin.read()
try:
  d=json.loads(l); print('$(basename $lib) $cfg', '| loss_ms %.3f | eff %.0f GB/s frac %.3f | status %s' % (d['roofline']['loss_ms_mean'], d['roofline']['achieved'], d['roofline']['frac'], d['status']))
except Exception as e: print('$lib FAILED', l[-300:])
"
  done
done
