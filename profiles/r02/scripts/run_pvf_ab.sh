# Forward-only exp2 MUFU/FMA split (npf of every 8 elements on the FMA pipe, backward all MUFU):
# variant library with kPoly entries 7 = {2, 0}, 8 = {1, 0}, 9 = {3, 0}; pv 0 = this build's default
O=gpurun_out/pvf_ab; mkdir -p $O
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw --format=csv,noheader -lms 200 > $O/clocks.csv &
SMI=$!
timeout 300 python profiles/r02/scripts/bwd_ab.py build_variants/libodpo_pvf.so tiny > /dev/null 2>&1
for i in 1 2 3; do
  for pv in 0 7 8 9; do
    timeout 300 python profiles/r02/scripts/bwd_ab.py build_variants/libodpo_pvf.so pythia llama --pv $pv 2>&1 | grep '^{'
  done
done | tee $O/pvf_ab.jsonl
kill $SMI
