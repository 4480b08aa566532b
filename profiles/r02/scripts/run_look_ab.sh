# Two-pass forward: rows decoded ahead by the engine's producer (kLook 1 = this build, 2, 3)
O=gpurun_out/look_ab; mkdir -p $O
timeout 300 python profiles/r02/scripts/bwd_ab.py main tiny > /dev/null 2>&1
for i in 1 2 3; do
  for L in main build_variants/libodpo_look2.so build_variants/libodpo_look3.so; do
    timeout 300 python profiles/r02/scripts/bwd_ab.py $L pythia rho llama 2>&1 | grep '^{'
  done
done | tee $O/look_ab.jsonl
