"""NEXT-2 forward A/B: odpo_lmhead_seq_logprobs on the Pythia / Rho / LLaMA heads vs cuBLAS's
bf16 GEMM alone, optionally against another libodpo build (argv[1])."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2410_18252_b200 as odpo  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1] != "default":
    odpo.LIB_PATH = os.path.abspath(sys.argv[1])


def t(fn, reps=7):
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


res = {"lib": sys.argv[1] if len(sys.argv) > 1 else "default"}
for name, (B, T, d, V) in {"pythia": (512, 53, 2560, 50304), "rho": (256, 512, 2048, 32000),
                           "llama": (128, 1024, 4096, 128256)}.items():
    g = torch.Generator(device="cuda").manual_seed(0)
    hid = (torch.randint(-32, 32, (B, T, d), device="cuda", generator=g).float() / 32).to(torch.bfloat16)
    Wh = (torch.randint(-32, 32, (V, d), device="cuda", generator=g).float() / 256).to(torch.bfloat16)
    tok = torch.randint(0, V, (B, T), device="cuda", generator=g, dtype=torch.int32)
    msk = torch.ones((B, T), dtype=torch.uint8, device="cuda")
    f = t(lambda: odpo.lmhead_seq_logprobs(hid, Wh, tok, msk))
    c = t(lambda: torch.matmul(hid.view(B * T, d), Wh.t()))
    fl = 2.0 * B * T * d * V
    res[name] = {"fused_ms": f, "fused_tflops": fl / f / 1e9, "cublas_ms": c, "cublas_tflops": fl / c / 1e9}
    del hid, Wh
    torch.cuda.empty_cache()
print(json.dumps(res), flush=True)
