#!/bin/bash
# FUSED (scaled dlogits) on geometry-1 variants: one CTA per SM, deep TMA ring, fewer rows in
# flight -> shorter dispatch-to-pair-completion latency -> backward re-read from L2?
# usage: profiles/tune_geo1.sh "cfg ..." ; reads build_variants/libodpo_g1_*.so
CFGS=${1:-"pythia rho"}
line() {
  python -c "
import json,sys
l=sys.stdin.read()
try:
  d=json.loads(l.strip().splitlines()[-1]); print('$1', '| loss_ms %.3f | eff %.0f GB/s frac %.3f | status %s' % (d['roofline']['loss_ms_mean'], d['roofline']['achieved'], d['roofline']['frac'], d['status']))
except Exception as e: print('$1 FAILED', l[-300:])
"
}
for cfg in $CFGS; do
  timeout 200 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux 2>&1 | line "$cfg default"
  for so in build_variants/libodpo_g1_*.so; do
    v=$(basename $so .so)
    for extra in "" "--lag 2" "--lag 4" "--lookahead 0"; do
      ODPO_LIB=$so timeout 200 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux --schedule fused --engine 1 $extra 2>&1 | line "$cfg $v $extra"
    done
  done
done
