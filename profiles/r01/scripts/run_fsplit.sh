# Experiment: FUSED forward rows split into ODPO_FSPLIT vocabulary parts (work units)
mkdir -p gpurun_out; : > gpurun_out/fsplit.log
line() { python -c "
import json,sys
l=sys.stdin.read()
try:
  d=json.loads(l.strip().splitlines()[-1]); print('$1', '| loss_ms %.3f | frac %.3f | status %s | loss %.10f' % (d['roofline']['loss_ms_mean'], d['roofline']['frac'], d['status'], d['loss']))
except Exception as e: print('$1 FAILED', l[-300:])
" >> gpurun_out/fsplit.log; }
ODPO_LIB=build_variants/libodpo_fs4.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "loss_parity_small and fused or self_consistency and fused or inplace and fused" > gpurun_out/fsplit_tests.log 2>&1; echo rc=$? >> gpurun_out/fsplit_tests.log
for cfg in pythia rho; do
  timeout 200 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux 2>&1 | line "$cfg default"
  for h in 2 4 7; do for lag in 0 8 24; do ODPO_LIB=build_variants/libodpo_fs$h.so timeout 200 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux --schedule fused --lag $lag 2>&1 | line "$cfg fs$h lag$lag"; done; done
done
