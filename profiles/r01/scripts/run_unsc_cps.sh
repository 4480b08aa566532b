# factored gradient: CTAs per SM (reuse distance of the backward re-read vs parallelism)
mkdir -p gpurun_out; : > gpurun_out/unsc_cps.log
line() { python -c "
import json,sys
l=sys.stdin.read()
try:
  d=json.loads(l.strip().splitlines()[-1]); print('$1', '| loss_ms %.3f | frac %.3f | status %s' % (d['roofline']['loss_ms_mean'], d['roofline']['frac'], d['status']))
except Exception as e: print('$1 FAILED', l[-300:])
" >> gpurun_out/unsc_cps.log; }
for cfg in pythia rho llama; do for c in 0 2 3; do timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux --gradient unscaled --ctas-per-sm $c 2>&1 | line "$cfg unscaled cps$c"; done; done
for cfg in pythia rho; do for c in 2 3; do timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux --loss rloo --ctas-per-sm $c 2>&1 | line "$cfg rloo cps$c"; done; done
