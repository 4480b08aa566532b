# interleaved repeats: unfused (cuBLAS) vs chunked vs recompute on the Pythia head
for i in 1 2 3; do
  timeout 600 python profiles/r02/lmhead_grad_bench.py --quick 2>&1 | tail -1
done
