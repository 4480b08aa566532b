#!/bin/bash
# quick sweep of schedule / exp2 split / lag on one workload; prints compact lines
CFG=${1:-pythia}
shift
VARIANTS=${@:-"--schedule two_pass|--exp2-split 0|--exp2-split 2|--exp2-split 6|--lag 2|--lag 8|--ctas-per-sm 1"}
IFS='|' read -ra ARR <<< "$VARIANTS"
for args in "${ARR[@]}"; do
  timeout 120 python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu --no-e2e $args 2>&1 | tail -1 | python -c "
import json,sys
l=sys.stdin.read()
try:
  d=json.loads(l); print('$args', '| pairs/s %.0f | loss_ms %.3f | eff %.0f GB/s frac %.3f | ref_ms %.3f (%.0f GB/s) | clk %s | status %s' % (d['value'], d['roofline']['loss_ms_mean'], d['roofline']['achieved'], d['roofline']['frac'], d['ref_pass_ms'], d['ref_pass_gbs'], d['clocks']['sm_mhz'], d['status']))
except Exception as e: print('$args FAILED', l[-300:])
"
done
