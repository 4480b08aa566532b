#!/bin/bash
# compute-sanitizer tools over every entry point (small shapes)
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
      python profiles/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? : $(grep -E 'ERROR SUMMARY|sanitize run ok' gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done
