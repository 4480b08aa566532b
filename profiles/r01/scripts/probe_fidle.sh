#!/bin/bash
for v in Gdbg FIdbg; do
  ODPO_LIB=$PWD/build_variants/libodpo_$v.so timeout 60 python profiles/prof_kernels.py --config pythia --variants fused:0 --reps 2 2>&1 | grep -E "LEAD|Error" | tail -2
done
for lib in default build_variants/libodpo_FI.so; do
  if [ "$lib" = default ]; then L=""; else L="ODPO_LIB=$PWD/$lib"; fi
  for cfg in pythia rho; do
  env $L timeout 120 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux --schedule fused 2>&1 | tail -1 | python -c "
import json,sys
l=sys.stdin.read()
try:
  d=json.loads(l); print('$(basename $lib) $cfg', '| loss_ms %.3f | eff %.0f GB/s frac %.3f | status %s' % (d['roofline']['loss_ms_mean'], d['roofline']['achieved'], d['roofline']['frac'], d['status']))
except Exception as e: print('$lib FAILED', l[-300:])
"
  done
  env $L ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_engine" -c 1 --csv python profiles/prof_kernels.py --config pythia --variants fused:0 --reps 1 2>/dev/null | grep k_engine | awk -F'","' '{print $(NF-2)" "$NF}'
done
