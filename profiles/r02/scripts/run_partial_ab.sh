# Partial-chunk batches (mr_partial) vs the padded full batch (ODPO_PARTIAL_OLD=1): the scaled
# call (two-pass) and the factored call, interleaved processes
O=gpurun_out/partial_ab; mkdir -p $O
timeout 300 python profiles/r02/scripts/bwd_ab.py main tiny > /dev/null 2>&1   # warm the box
for i in 1 2 3; do
  for L in main build_variants/libodpo_pold.so; do
    timeout 300 python profiles/r02/scripts/bwd_ab.py $L pythia rho llama 2>&1 | grep '^{'
    if [ $L = main ]; then timeout 300 python profiles/r02/scripts/split_ab.py pythia rho llama 2>&1 | grep '^{' | sed 's/^{/{"lib": "main", /';
    else timeout 300 python profiles/r02/scripts/split_ab.py $L pythia rho llama 2>&1 | grep '^{' | sed 's/^{/{"lib": "pold", /'; fi
  done
done | tee $O/partial_ab.jsonl
