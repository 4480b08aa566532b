# LLaMA-head forward raster group (ODPO_LMH_G = 2 x the 256-row pair-blocks per group): DRAM /
# L2 traffic per launch (ncu metrics) and the sustained clock / time per call (power probe)
O=gpurun_out/raster; mkdir -p $O
for g in 24 32 48 64 128; do
  L=build_variants/libodpo_lmhg$g.so; [ $g = 64 ] && L=paper_2410_18252_b200/libodpo.so
  timeout 300 python profiles/r02/next2/scripts/head_once.py $L > /dev/null 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:k_lmhead_fwd2 -s 2 -c 1 --csv python profiles/r02/next2/scripts/head_once.py $L 2>/dev/null | grep -v "^==" | sed "s/^/G$g,/" >> $O/ncu.csv
  timeout 300 python profiles/r02/next2/scripts/power_probe.py $L 2>&1 | grep odpo | sed "s/^{/{\"G\": $g, /" >> $O/probe.jsonl
done
cat $O/ncu.csv | grep -v '"ID"' | awk -F'","' '{print $1, $(NF-2), $NF}'; cat $O/probe.jsonl
