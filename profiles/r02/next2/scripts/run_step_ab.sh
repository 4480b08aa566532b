timeout 300 python profiles/r02/next2/scripts/step_ab.py main > /dev/null 2>&1   # warm the box
for i in 1 2 3 4 5 6 7 8; do
  timeout 300 python profiles/r02/next2/scripts/step_ab.py main 2>&1 | tail -1
  timeout 300 python profiles/r02/next2/scripts/step_ab.py build_variants/libodpo_fwdpass.so 2>&1 | tail -1
done | tee gpurun_out/step_ab.jsonl
