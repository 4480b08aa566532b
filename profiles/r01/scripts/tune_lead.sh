#!/bin/bash
for lib in G K C; do
  for lag in 3 4 6 8 12 0; do
    ODPO_LIB=$PWD/build_variants/libodpo_$lib.so timeout 60 python bench.py --config pythia --steps 10 --warmup 3 --no-cpu --no-e2e --lag $lag 2>&1 | tail -1 | python -c "
import json,sys
l=sys.stdin.read()
try:
  d=json.loads(l); print('$lib lag $lag', '| pairs/s %.0f | loss_ms %.3f | eff %.0f GB/s | ref_ms %.3f' % (d['value'], d['roofline']['loss_ms_mean'], d['roofline']['achieved'], d['ref_pass_ms']))
except Exception as e: print('$lib $lag FAILED', l[-300:])
"
  done
done
