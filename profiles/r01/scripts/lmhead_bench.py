"""NEXT-2 timing: fused LM-head log-probs (tcgen05, logits never written) vs the unfused
path (cuBLAS bf16 GEMM writing logits + odpo.seq_logprobs reading them).  Pythia TLDR shape
by default: rows = 256 pairs x 2 x 53, d = 2560, V = 50304.  Prints one JSON line."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2410_18252_b200 as odpo  # noqa: E402
import synth  # noqa: E402

B, T, d, V = (int(x) for x in sys.argv[1:5]) if len(sys.argv) > 4 else (512, 53, 2560, 50304)
steps = 10
g = torch.Generator(device="cuda").manual_seed(0)
hid = (torch.randint(-32, 32, (B, T, d), device="cuda", generator=g).float() / 32).to(torch.bfloat16)
W = (torch.randint(-32, 32, (V, d), device="cuda", generator=g).float() / 256).to(torch.bfloat16)
tok = torch.randint(0, V, (B, T), device="cuda", generator=g, dtype=torch.int32)
mask = torch.ones((B, T), dtype=torch.uint8, device="cuda")
flops = 2.0 * B * T * d * V


def timeit(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev]))


fused_ms = timeit(lambda: odpo.lmhead_seq_logprobs(hid, W, tok, mask))
seq_f = odpo.lmhead_seq_logprobs(hid, W, tok, mask)[0]
gemm_ms = timeit(lambda: torch.matmul(hid.view(B * T, d), W.t()))
logits = torch.matmul(hid.view(B * T, d), W.t()).view(B, T, V)
seq_ms = timeit(lambda: odpo.seq_logprobs(logits, tok, mask))
seq_u = odpo.seq_logprobs(logits, tok, mask)
torch.cuda.synchronize()
# the unfused path rounds the logits to bf16 before the log-softmax; the fused path does not
rel = float(((seq_f.double() - seq_u.double()).abs() / seq_u.double().abs().clamp_min(1)).max())
peaks = {}
try:
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
except Exception:
    pass
print(json.dumps({"shape": [B, T, d, V], "fused_ms": fused_ms, "fused_tflops": flops / fused_ms / 1e9,
                  "cublas_gemm_ms": gemm_ms, "cublas_tflops": flops / gemm_ms / 1e9,
                  "seq_logprobs_ms": seq_ms, "unfused_ms": gemm_ms + seq_ms,
                  "speedup_vs_unfused": (gemm_ms + seq_ms) / fused_ms,
                  "max_rel_seq_diff_vs_bf16_logits": rel, "measured_peaks": peaks}))
