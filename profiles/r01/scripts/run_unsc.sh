#!/bin/bash
# unscaled-gradient path: GPU tests, then bench lines for pythia / rho / llama both forms
set -x
timeout 900 python -m pytest tests/test_gpu_unscaled.py -q -x --timeout 300 --timeout-method thread 2>&1 | tail -5
for cfg in pythia rho llama; do
  timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e --gradient unscaled 2>gpurun_out/unsc_$cfg.err | tail -1 > gpurun_out/unsc_$cfg.json
  python -c "
import json; d=json.load(open('gpurun_out/unsc_$cfg.json'))
r=d['roofline']; a=d['aux_gradient_form']
print('$cfg unscaled: loss_ms %.3f eff %.0f frac %.3f | scaled: loss_ms %.3f frac %.3f | status %s/%s' % (r['loss_ms_mean'], r['achieved'], r['frac'], a['loss_ms_mean'], a['frac'], d['status'], a['status']))
" || tail -5 gpurun_out/unsc_$cfg.err
done
