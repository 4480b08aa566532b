mkdir -p gpurun_out; : > gpurun_out/res_un2.log
line() { python -c "
import json,sys
l=sys.stdin.read()
try:
  d=json.loads(l.strip().splitlines()[-1]); print('$1', '| loss_ms %.3f | frac %.3f | status %s' % (d['roofline']['loss_ms_mean'], d['roofline']['frac'], d['status']))
except Exception as e: print('$1 FAILED', l[-300:])
" >> gpurun_out/res_un2.log; }
for cap in 0 1 2; do ODPO_LIB=build_variants/libodpo_fw8.so timeout 200 python bench.py --config pythia --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux --gradient unscaled --schedule resident --lookahead $cap 2>&1 | line "pythia unscaled resident FW8 cap$cap"; done
ODPO_LIB=build_variants/libodpo_fw8.so timeout 200 python bench.py --config pythia --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux --schedule resident 2>&1 | line "pythia scaled resident FW8 cap2"
