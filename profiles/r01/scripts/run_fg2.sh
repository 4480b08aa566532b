# RESIDENT with two forward warp groups (ODPO_RES_FGROUPS=2): parity (bit-identity with FUSED)
# and the factored-gradient / scaled timings
mkdir -p gpurun_out; : > gpurun_out/fg2.log
ODPO_LIB=build_variants/libodpo_fg2.so timeout 400 python -m pytest tests/test_gpu_unscaled.py tests/test_gpu_parity.py -q -k "resident or unscaled_parity_small or best_worst" > gpurun_out/fg2_tests.log 2>&1; echo rc=$? >> gpurun_out/fg2_tests.log
line() { python -c "
import json,sys
l=sys.stdin.read()
try:
  d=json.loads(l.strip().splitlines()[-1]); print('$1', '| loss_ms %.3f | frac %.3f | status %s' % (d['roofline']['loss_ms_mean'], d['roofline']['frac'], d['status']))
except Exception as e: print('$1 FAILED', l[-300:])
" >> gpurun_out/fg2.log; }
for cfg in pythia rho; do
  timeout 200 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux --gradient unscaled 2>&1 | line "$cfg unscaled engine"
  for cap in 0 1 2; do ODPO_LIB=build_variants/libodpo_fg2.so timeout 200 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux --gradient unscaled --schedule resident --lookahead $cap 2>&1 | line "$cfg unscaled resident FG2 cap$cap"; done
done
ODPO_LIB=build_variants/libodpo_fg2.so timeout 200 python bench.py --config pythia --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux --schedule resident 2>&1 | line "pythia scaled resident FG2 cap2"
