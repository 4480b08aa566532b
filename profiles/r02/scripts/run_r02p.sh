timeout 900 python -m pytest tests/test_gpu_unscaled.py tests/test_gpu_parity.py -q --timeout 300 -x 2>&1 | tail -3
ab() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', d['config']['workload'], 'loss_ms %.3f frac %.3f' % (r['loss_ms_mean'], r['frac']), d['clocks']['sm_mhz'], d['status'])"; }
for cfg in llama rho pythia; do
  for eng in -1 0 1 2; do
    for gap in 0 2; do
      timeout 300 python bench.py --config $cfg --gradient unscaled --steps 10 --warmup 3 --no-aux --no-e2e --no-cpu --engine $eng --row-gap $gap 2>/dev/null | ab ${cfg}_eng${eng}_gap$gap
    done
  done
done
