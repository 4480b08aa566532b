#!/bin/bash
# L2 reuse probe of the fused kernel: DRAM bytes and L2 hit rate per variant library
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for lib in default build_variants/libodpo_C2.so build_variants/libodpo_C4.so; do
  if [ "$lib" = default ]; then L=""; else L="ODPO_LIB=$PWD/$lib"; fi
  echo "== $lib"
  env $L ncu --metrics $M --clock-control none -k regex:"k_engine" -c 3 --csv python profiles/prof_kernels.py --config pythia --variants fused:0 --reps 1 2>/dev/null | grep -E "k_engine" | awk -F'","' '{print $5" | "$(NF-2)" "$(NF-1)" "$NF}' | tail -8
done
