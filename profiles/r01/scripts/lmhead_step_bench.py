"""NEXT-2 full learner step on the LM head (forward + DPO loss + backward to hidden and weight):
fused (logits never stored: lmhead_online_dpo_loss_fwd + lmhead_grad, logits recomputed in
row chunks) vs unfused (cuBLAS logits GEMM + odpo_online_dpo_loss_fwd_bwd writing dlogits +
two cuBLAS GEMMs).  Times and peak memory; Pythia TLDR shape by default."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2410_18252_b200 as odpo  # noqa: E402

P, T, d, V = (int(x) for x in sys.argv[1:5]) if len(sys.argv) > 4 else (256, 53, 2560, 50304)
chunk = int(sys.argv[5]) if len(sys.argv) > 5 else 8192
B = 2 * P
g = torch.Generator(device="cuda").manual_seed(0)
hid = (torch.randint(-32, 32, (B, T, d), device="cuda", generator=g).float() / 32).to(torch.bfloat16)
W = (torch.randint(-32, 32, (V, d), device="cuda", generator=g).float() / 256).to(torch.bfloat16)
tok = torch.randint(0, V, (B, T), device="cuda", generator=g, dtype=torch.int32)
mask = torch.ones((B, T), dtype=torch.uint8, device="cuda")
ref = torch.full((B,), -float(T) * 4.0, device="cuda")


def fused():
    out = odpo.lmhead_online_dpo_loss_fwd(hid, W, ref, tok, mask, 0.1)
    return odpo.lmhead_grad(hid, W, tok, out.row_lse, out.row_scale, chunk_rows=chunk)


def unfused():
    logits = torch.matmul(hid.view(B * T, d), W.t()).view(B, T, V)
    out = odpo.online_dpo_loss_fwd_bwd(logits, ref, tok, mask, 0.1, inplace=True)
    dl = out.dlogits.view(B * T, V)
    dh = torch.matmul(dl, W).float()
    dw = torch.matmul(dl.t(), hid.view(B * T, d)).float()
    return dh, dw


def timeit(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev])), (torch.cuda.max_memory_allocated() - base) / 1e9


f_ms, f_mem = timeit(fused)
u_ms, u_mem = timeit(unfused)
dhf, dwf = fused()
dhu, dwu = unfused()
torch.cuda.synchronize()
rel_h = float((dhf.reshape(-1, d) - dhu.reshape(-1, d)).norm() / dhu.norm())
rel_w = float((dwf - dwu).norm() / dwu.norm())
flops_fwd = 2.0 * B * T * d * V
print(json.dumps({"shape": [P, T, d, V], "chunk_rows": chunk, "fused_ms": f_ms, "fused_peak_extra_gb": f_mem,
                  "unfused_ms": u_ms, "unfused_peak_extra_gb": u_mem,
                  "fused_tflops_4gemm": 4 * flops_fwd / f_ms / 1e9, "unfused_tflops_3gemm": 3 * flops_fwd / u_ms / 1e9,
                  "rel_diff_dhidden": rel_h, "rel_diff_dweight": rel_w}))
