# Two-pass (AUTO) loss call: engine geometry and CTAs per SM of the forward, per config
O=gpurun_out/geo_sweep; mkdir -p $O
for cfg in pythia rho llama; do
  for g in "0 0" "0 3" "0 2" "1 0" "1 1"; do
    set -- $g
    timeout 600 python bench.py --config $cfg --no-aux --no-e2e --no-cpu --engine $1 --ctas-per-sm $2 --steps 10 2>/dev/null | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); r = d['roofline']
print(json.dumps({'config': '$cfg', 'engine': $1, 'cps': $2, 'loss_ms': r['loss_ms_mean'], 'frac': r['frac'], 'loss': d['loss'], 'clk': d['clocks']['sm_mhz']}))"
  done
done | tee $O/geo_sweep.jsonl
