ab() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', d['config']['workload'], 'loss_ms %.4f frac %.3f' % (r['loss_ms_mean'], r['frac']), d['gpu_launches'])"; }
for rep in 1 2; do
for sch in auto fused wave two_pass; do
  timeout 300 python bench.py --config tiny --schedule $sch --steps 20 --warmup 5 --no-aux --no-e2e --no-cpu 2>/dev/null | ab tiny_$sch
done
done
