# A/B of the split-row backward configurations (profiles/r02/scripts/bwd_ab.py), interleaved
O=gpurun_out/bwd_ab2; mkdir -p $O
timeout 300 python profiles/r02/scripts/bwd_ab.py main tiny > /dev/null 2>&1   # warm the box
for i in 1 2 3; do
  for L in main build_variants/libodpo_bwd-1.so build_variants/libodpo_bwd6.so build_variants/libodpo_bwd7.so; do
    timeout 300 python profiles/r02/scripts/bwd_ab.py $L pythia rho llama 2>&1 | grep '^{'
  done
done | tee $O/bwd_ab.jsonl
