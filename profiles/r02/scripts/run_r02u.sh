ab() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', d['config']['workload'], 'loss_ms %.3f frac %.3f' % (r['loss_ms_mean'], r['frac']), d['clocks']['sm_mhz'])"; }
for rep in 1 2; do
for cfg in llama pythia rho; do
  timeout 300 python bench.py --config $cfg --gradient unscaled --steps 10 --warmup 3 --no-aux --no-e2e --no-cpu 2>/dev/null | ab ${cfg}_ug100
  for pct in 60 75 87; do
    timeout 300 python bench.py --config $cfg --gradient unscaled --steps 10 --warmup 3 --no-aux --no-e2e --no-cpu --lib build_variants/libodpo_ug$pct.so 2>/dev/null | ab ${cfg}_ug$pct
  done
done
done
