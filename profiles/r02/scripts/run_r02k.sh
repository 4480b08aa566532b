O=gpurun_out/r02k; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x --timeout 120 -k "psync" 2>&1 | tail -25
ab() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', d['config']['workload'], 'loss_ms %.3f frac %.3f' % (r['loss_ms_mean'], r['frac']), d['clocks']['sm_mhz'], d['status'])"; }
timeout 120 python bench.py --config pythia --steps 20 --warmup 5 --no-aux --no-e2e --no-cpu 2>/dev/null | ab fused
for lag in 1 2 4 8 12; do
  timeout 120 python bench.py --config pythia --steps 20 --warmup 5 --no-aux --no-e2e --no-cpu --schedule psync --lag $lag 2>&1 | tail -1 | ab psync_lag$lag
done
timeout 120 python bench.py --config tiny --steps 20 --warmup 5 --no-aux --no-e2e --no-cpu --schedule psync --lag 2 2>&1 | tail -1 | ab psync_tiny
timeout 300 ncu --set full --clock-control none -k regex:"k_psync" -s 3 -c 1 -o /tmp/ps -f python bench.py --config pythia --steps 1 --warmup 3 --no-e2e --no-cpu --no-aux --schedule psync --lag 4 > /dev/null 2>&1
python profiles/summarize_ncu.py r02k_psync pythia psync "" /tmp/ps.ncu-rep 2>&1 | grep -E "DRAM|duration|L2 hit|issue|MUFU|warps" 
