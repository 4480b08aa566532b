O=gpurun_out/r02j; mkdir -p $O
timeout 900 python -m pytest tests/test_lmhead.py -q -x --timeout 600 2>&1 | tail -2
timeout 600 python profiles/r02/lmhead_grad_bench.py --quick 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_gemm|k_lmhead_fwd2" --csv --log-file $O/grad_launches.csv python profiles/r02/lmhead_grad_bench.py --quick > /dev/null 2>&1
python profiles/summarize_ncu.py r02j_grad pythia grad $O/grad_launches.csv 2>&1 | grep "k_"
ab() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', d['config']['workload'], 'loss_ms %.3f frac %.3f' % (r['loss_ms_mean'], r['frac']), d['clocks']['sm_mhz'])"; }
for cps in 0 1; do
  timeout 300 python bench.py --config llama --gradient unscaled --steps 10 --warmup 3 --no-aux --no-e2e --no-cpu --ctas-per-sm $cps 2>/dev/null | ab llama_geo1_cps$cps
done
timeout 300 python bench.py --config llama --gradient unscaled --steps 10 --warmup 3 --no-aux --no-e2e --no-cpu --engine 0 2>/dev/null | ab llama_geo0
for cps in 0 2 3; do
  timeout 300 python bench.py --config pythia --gradient unscaled --steps 20 --warmup 5 --no-aux --no-e2e --no-cpu --ctas-per-sm $cps 2>/dev/null | ab pythia_geo0_cps$cps
done
timeout 300 python bench.py --config pythia --gradient unscaled --steps 20 --warmup 5 --no-aux --no-e2e --no-cpu --engine 1 2>/dev/null | ab pythia_geo1
timeout 300 python bench.py --config rho --gradient unscaled --steps 20 --warmup 5 --no-aux --no-e2e --no-cpu 2>/dev/null | ab rho_auto
timeout 300 python bench.py --config rho --gradient unscaled --steps 20 --warmup 5 --no-aux --no-e2e --no-cpu --engine 1 2>/dev/null | ab rho_geo1
