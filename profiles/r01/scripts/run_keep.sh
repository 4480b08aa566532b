# Experiment: forward rows' L2 policy = evict_last on a fraction f of the lines (rest evict_first)
mkdir -p gpurun_out; : > gpurun_out/keep.log
line() { python -c "
import json,sys
l=sys.stdin.read()
try:
  d=json.loads(l.strip().splitlines()[-1]); print('$1', '| loss_ms %.3f | frac %.3f | status %s' % (d['roofline']['loss_ms_mean'], d['roofline']['frac'], d['status']))
except Exception as e: print('$1 FAILED', l[-300:])
" >> gpurun_out/keep.log; }
for cfg in pythia rho; do
  timeout 200 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux 2>&1 | line "$cfg default"
  for f in 10 20 30 50; do ODPO_LIB=build_variants/libodpo_keep$f.so timeout 200 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux 2>&1 | line "$cfg keep$f"; done
done
ODPO_LIB=build_variants/libodpo_keep20.so timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_engine -s 4 -c 2 --csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-aux > gpurun_out/keep_ncu.csv 2>&1
