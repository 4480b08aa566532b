# exp2_split (MUFU / FMA-polynomial split) sweep of the scaled loss call (AUTO = TWO_PASS)
O=gpurun_out/pv_ab; mkdir -p $O
timeout 300 python profiles/r02/scripts/bwd_ab.py main tiny > /dev/null 2>&1   # warm the box
for i in 1 2; do
  for pv in 0 1 2 3 4 5 6; do
    timeout 300 python profiles/r02/scripts/bwd_ab.py main pythia rho llama --pv $pv 2>&1 | grep '^{'
  done
done | tee $O/pv_ab.jsonl
