"""A/B of the chunked NEXT-2 learner step (Pythia head): this build vs a variant library given
as argv[1] (e.g. build_variants/libodpo_fwdpass.so = the round-2 step with the loss forward
pass).  Prints one JSON line: medians of 7 calls, the unfused (cuBLAS) step beside it."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(
    os.path.abspath(__file__)))))))
import paper_2410_18252_b200 as odpo  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1] != "main":
    odpo.LIB_PATH = os.path.abspath(sys.argv[1])
B, T, d, V = 512, 53, 2560, 50304
g = torch.Generator(device="cuda").manual_seed(0)
hid = (torch.randint(-32, 32, (B, T, d), device="cuda", generator=g).float() / 32).to(torch.bfloat16)
Wh = (torch.randint(-32, 32, (V, d), device="cuda", generator=g).float() / 256).to(torch.bfloat16)
tok = torch.randint(0, V, (B, T), device="cuda", generator=g, dtype=torch.int32)
msk = torch.ones((B, T), dtype=torch.uint8, device="cuda")
ref = torch.full((B,), -4.0 * T, device="cuda")


def t(fn, reps=15):
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


def unfused():
    lg = torch.matmul(hid.view(B * T, d), Wh.t()).view(B, T, V)
    oo = odpo.online_dpo_loss_fwd_bwd(lg, ref, tok, msk, 0.1, inplace=True)
    dl = oo.dlogits.view(B * T, V)
    return torch.matmul(dl, Wh), torch.matmul(dl.t(), hid.view(B * T, d))


out = {"lib": sys.argv[1] if len(sys.argv) > 1 else "main",
       "chunked_ms": t(lambda: odpo.lmhead_dpo_step(hid, Wh, ref, tok, msk, 0.1)),
       "unfused_ms": t(unfused)}
print(json.dumps(out), flush=True)
