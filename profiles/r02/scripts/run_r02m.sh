# round 2: compute-sanitizer over every entry point (new: seq_ppl, VP put/wait, tcgen05 GEMMs),
# and one ncu --set full capture of each backward GEMM
O=gpurun_out/r02m; mkdir -p $O
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
      python profiles/sanitize_run.py > $O/sanitize_$tool.log 2>&1
  echo "$tool rc=$? : $(grep -E 'ERROR SUMMARY|sanitize run ok' $O/sanitize_$tool.log | tr '\n' ' ')"
done
timeout 600 ncu --set full --clock-control none -k regex:"k_gemm_tn2|k_lmhead_fwd2" -s 3 -c 3 -o /tmp/g -f python profiles/r02/lmhead_grad_bench.py --quick > /dev/null 2>&1
python profiles/summarize_ncu.py r02m_gemm pythia gemm "" /tmp/g.ncu-rep > $O/gemm_full.md 2>&1
cat $O/gemm_full.md | grep -vE "^$" | head -60
ncu -i /tmp/g.ncu-rep --page details --csv 2>/dev/null | grep -iE "tensor|Stall|Pipe" | head -40 > $O/gemm_details.csv
head -40 $O/gemm_details.csv
