# RESIDENT: forward-queue bound x L2 cap
mkdir -p gpurun_out; : > gpurun_out/res_fq.log
line() { python -c "
import json,sys
l=sys.stdin.read()
try:
  d=json.loads(l.strip().splitlines()[-1]); print('$1', '| loss_ms %.3f | frac %.3f | status %s' % (d['roofline']['loss_ms_mean'], d['roofline']['frac'], d['status']))
except Exception as e: print('$1 FAILED', l[-300:])
" >> gpurun_out/res_fq.log; }
for q in 1 2; do for cap in 2 4 6; do ODPO_LIB=build_variants/libodpo_fq$q.so timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux --schedule resident --lookahead $cap 2>&1 | line "fq$q cap$cap"; done; done
