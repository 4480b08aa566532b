# Pythia head learner step: this build vs the dynamic order for the head-forward kernels too
O=gpurun_out/step_ab2; mkdir -p $O
timeout 300 python profiles/r02/next2/scripts/step_ab.py main > /dev/null 2>&1
for i in 1 2 3 4 5 6; do
  timeout 300 python profiles/r02/next2/scripts/step_ab.py main 2>&1 | tail -1
  timeout 300 python profiles/r02/next2/scripts/step_ab.py build_variants/libodpo_dynall.so 2>&1 | tail -1
done | tee $O/step_ab.jsonl
