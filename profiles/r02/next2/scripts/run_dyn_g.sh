# Dynamic tile order: raster group sweep (sustained clock / time per LLaMA- and Pythia-head forward)
O=gpurun_out/dyn_g; mkdir -p $O
for g in 24 32 48 64 96; do
  L=build_variants/libodpo_dg$g.so; [ $g = 64 ] && L=paper_2410_18252_b200/libodpo.so
  timeout 300 python profiles/r02/next2/scripts/power_probe.py $L 2>&1 | grep odpo | sed "s/^{/{\"G\": $g, /" >> $O/probe.jsonl
done
cat $O/probe.jsonl
