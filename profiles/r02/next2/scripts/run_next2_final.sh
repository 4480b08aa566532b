# NEXT-2 after the dynamic tile order: parity, chunked vs unfused steps (Pythia: interleaved
# process pairs; LLaMA: the grad bench twice), head forward power probe
O=gpurun_out/next2_final; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -2 > $O/gpu_tests.log; cat $O/gpu_tests.log
for i in 1 2 3 4; do timeout 300 python profiles/r02/next2/scripts/step_ab.py main 2>&1 | tail -1; done > $O/step_ab_pythia.jsonl
for i in 1 2; do timeout 600 python profiles/r02/lmhead_grad_bench.py llama --quick 2>&1 | tail -1; done > $O/grad_llama.jsonl
timeout 300 python profiles/r02/lmhead_grad_bench.py --quick 2>&1 | tail -1 > $O/grad_pythia.jsonl
timeout 300 python profiles/r02/next2/scripts/power_probe.py 2>&1 | tail -4 > $O/probe.jsonl
cat $O/*.jsonl
