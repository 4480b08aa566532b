"""NEXT-2 backward timing on the Pythia-2.8B head (512 x 53 rows, d 2560, V 50304): the whole
odpo_lmhead_grad call for several chunk sizes, and the fused / unfused learner steps."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2410_18252_b200 as odpo  # noqa: E402

for _a in sys.argv[1:]:
    if _a.endswith(".so"):   # a variant build (A/B)
        odpo.LIB_PATH = os.path.abspath(_a)


def t(fn, reps=5):
    for _ in range(2):
        fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    torch.cuda.synchronize()
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in ev)[reps // 2]


B, T, d, V = 512, 53, 2560, 50304
if "llama" in sys.argv:
    B, T, d, V = 128, 1024, 4096, 128256
g = torch.Generator(device="cuda").manual_seed(0)
hid = (torch.randint(-32, 32, (B, T, d), device="cuda", generator=g).float() / 32).to(torch.bfloat16)
Wh = (torch.randint(-32, 32, (V, d), device="cuda", generator=g).float() / 256).to(torch.bfloat16)
tok = torch.randint(0, V, (B, T), device="cuda", generator=g, dtype=torch.int32)
msk = torch.ones((B, T), dtype=torch.uint8, device="cuda")
ref = torch.full((B,), -4.0 * T, device="cuda")
o = odpo.lmhead_online_dpo_loss_fwd(hid, Wh, ref, tok, msk, 0.1)
flops = 2.0 * B * T * d * V
res = {"shape": [B, T, d, V], "fwd_ms": t(lambda: odpo.lmhead_online_dpo_loss_fwd(hid, Wh, ref, tok, msk, 0.1))}
CHUNKS = (None,) if "--quick" in sys.argv else (None, 4736, 9472, 18944, 27136)
for ch in CHUNKS:
    if ch is not None and ch > B * T:
        continue
    ms = t(lambda: odpo.lmhead_grad(hid, Wh, tok, o.row_lse, o.row_scale, chunk_rows=ch))
    res[f"grad_ms_chunk_{ch}"] = ms
    res[f"grad_tflops_chunk_{ch}"] = 3 * flops / ms / 1e9
res["step_chunked_ms"] = t(lambda: odpo.lmhead_dpo_step(hid, Wh, ref, tok, msk, 0.1))


def recompute_step():
    oo = odpo.lmhead_online_dpo_loss_fwd(hid, Wh, ref, tok, msk, 0.1)
    return odpo.lmhead_grad(hid, Wh, tok, oo.row_lse, oo.row_scale)


res["step_recompute_ms"] = t(recompute_step)


def unfused():
    lg = torch.matmul(hid.view(B * T, d), Wh.t()).view(B, T, V)
    oo = odpo.online_dpo_loss_fwd_bwd(lg, ref, tok, msk, 0.1, inplace=True)
    dl = oo.dlogits.view(B * T, V)
    return torch.matmul(dl, Wh), torch.matmul(dl.t(), hid.view(B * T, d))


res["step_unfused_ms"] = t(unfused)
gemm = t(lambda: torch.matmul(hid.view(B * T, d), Wh.t()))
res["cublas_logits_gemm_ms"] = gemm
print(json.dumps(res), flush=True)
