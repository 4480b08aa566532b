# RESIDENT factored gradient: parity + bench vs the row engine (Pythia, Rho), cap sweep
mkdir -p gpurun_out; : > gpurun_out/res_un.log
timeout 600 python -m pytest tests/test_gpu_unscaled.py -x -q > gpurun_out/res_un_tests.log 2>&1; echo rc=$? >> gpurun_out/res_un_tests.log
line() { python -c "
import json,sys
l=sys.stdin.read()
try:
  d=json.loads(l.strip().splitlines()[-1]); print('$1', '| loss_ms %.3f | frac %.3f | status %s' % (d['roofline']['loss_ms_mean'], d['roofline']['frac'], d['status']))
except Exception as e: print('$1 FAILED', l[-300:])
" >> gpurun_out/res_un.log; }
for cfg in pythia rho; do
  timeout 200 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux --gradient unscaled 2>&1 | line "$cfg unscaled engine"
  for cap in 0 1 2 4; do timeout 200 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux --gradient unscaled --schedule resident --lookahead $cap 2>&1 | line "$cfg unscaled resident cap$cap"; done
done
