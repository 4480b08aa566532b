# NEXT-4 short shard rows: CTA-per-row partials + one-batch backward pieces (main) vs round 2's
# warp-per-row kernels (build_variants/libodpo_vpwarp.so), interleaved
O=gpurun_out/vp_ab; mkdir -p $O
for i in 1 2; do
  for cfg in pythia rho llama; do for W in 2 8; do
    for L in main build_variants/libodpo_vpwarp.so; do
      X=""; [ $L != main ] && X="--lib $L"
      timeout 300 python profiles/vp_bench.py --config $cfg --W $W $X 2>&1 | tail -1 | sed "s#^{#{\"lib\": \"$L\", #"
      timeout 300 python profiles/vp_bench.py --config $cfg --W $W --put $X 2>&1 | tail -1 | sed "s#^{#{\"lib\": \"$L\", #"
    done
  done; done
done | tee $O/vp_ab.jsonl
