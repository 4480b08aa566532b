timeout 600 python -m pytest tests/test_gpu_unscaled.py -q --timeout 300 -x -k "engine2 or 2-0" 2>&1 | tail -3
ab() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', d['config']['workload'], 'loss_ms %.3f frac %.3f' % (r['loss_ms_mean'], r['frac']), d['clocks']['sm_mhz'], d['status'])"; }
for cfg in llama rho pythia; do
  for eng in -1 2; do
    timeout 300 python bench.py --config $cfg --gradient unscaled --steps 10 --warmup 3 --no-aux --no-e2e --no-cpu --engine $eng 2>/dev/null | ab ${cfg}_unscaled_eng$eng
  done
done
timeout 300 python bench.py --config llama --steps 10 --warmup 3 --no-aux --no-e2e --no-cpu --engine 2 2>/dev/null | ab llama_scaled_eng2
timeout 600 ncu --set full --clock-control none -k regex:"k_engine" -s 4 -c 1 -o /tmp/u2 -f python bench.py --config llama --steps 1 --warmup 3 --no-e2e --no-cpu --no-aux --gradient unscaled --engine 2 > /dev/null 2>&1
python profiles/summarize_ncu.py r02o_llama_unscaled_eng2 llama unscaled_eng2 "" /tmp/u2.ncu-rep 2>&1 | grep -E "DRAM|duration|L2 hit"
