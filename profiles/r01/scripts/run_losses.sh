#!/bin/bash
# bench lines of the App B losses next to Online DPO (pythia, rho, llama)
mkdir -p gpurun_out/losses
for cfg in pythia rho llama; do
  for loss in dpo rloo copg prox_rloo sft; do
    timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux --loss $loss \
      > gpurun_out/losses/${cfg}_${loss}.json 2> gpurun_out/losses/${cfg}_${loss}.err
    python -c "
import json; d=json.load(open('gpurun_out/losses/${cfg}_${loss}.json')); r=d['roofline']
print('$cfg $loss | pairs/s %.0f | loss_ms %.3f | eff %.0f GB/s frac %.3f | status %s | loss %.5f' % (d['value'], r['loss_ms_mean'], r['achieved'], r['frac'], d['status'], d['loss']))
" || tail -3 gpurun_out/losses/${cfg}_${loss}.err
  done
done
