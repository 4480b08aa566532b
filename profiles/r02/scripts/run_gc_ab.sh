# (1) kernel parameters as __grid_constant__ (no per-thread local copy of LossArgs in the
# engines that call the pair reduction) and (2) 20 KB engine chunks, vs this build
O=gpurun_out/gc_ab; mkdir -p $O
timeout 300 python profiles/r02/scripts/bwd_ab.py main tiny > /dev/null 2>&1   # warm the box
for i in 1 2 3; do
  for L in main build_variants/libodpo_gc.so build_variants/libodpo_c20a.so build_variants/libodpo_c20b.so; do
    timeout 300 python profiles/r02/scripts/bwd_ab.py $L pythia rho llama 2>&1 | grep '^{'
    if [ $L = main ]; then timeout 300 python profiles/r02/scripts/split_ab.py pythia rho llama 2>&1 | grep '^{' | sed 's/^{/{"lib": "main", /';
    else timeout 300 python profiles/r02/scripts/split_ab.py $L pythia rho llama 2>&1 | grep '^{' | sed "s#^{#{\"lib\": \"$L\", #"; fi
  done
done | tee $O/gc_ab.jsonl
