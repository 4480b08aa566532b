ab() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', d['config']['workload'], 'loss_ms %.4f frac %.3f' % (r['loss_ms_mean'], r['frac']), d['gpu_launches'], d['clocks']['sm_mhz'])"; }
for cfg in tiny pythia rho llama; do
for sch in auto fused two_pass; do
  timeout 300 python bench.py --config $cfg --schedule $sch --steps 10 --warmup 3 --no-aux --no-e2e --no-cpu 2>/dev/null | ab ${cfg}_$sch
done
done
timeout 600 python -m pytest tests/test_gpu_safety.py tests/test_gpu_parity.py -q --timeout 300 -x 2>&1 | tail -2
