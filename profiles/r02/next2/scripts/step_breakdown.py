"""One chunked NEXT-2 learner step and one unfused step (Pythia head), after warm-up, for an
ncu launch list (per-kernel durations of each phase)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(
    os.path.abspath(__file__)))))))
import paper_2410_18252_b200 as odpo  # noqa: E402

B, T, d, V = 512, 53, 2560, 50304
g = torch.Generator(device="cuda").manual_seed(0)
hid = (torch.randint(-32, 32, (B, T, d), device="cuda", generator=g).float() / 32).to(torch.bfloat16)
Wh = (torch.randint(-32, 32, (V, d), device="cuda", generator=g).float() / 256).to(torch.bfloat16)
tok = torch.randint(0, V, (B, T), device="cuda", generator=g, dtype=torch.int32)
msk = torch.ones((B, T), dtype=torch.uint8, device="cuda")
ref = torch.full((B,), -4.0 * T, device="cuda")


def unfused():
    lg = torch.matmul(hid.view(B * T, d), Wh.t()).view(B, T, V)
    oo = odpo.online_dpo_loss_fwd_bwd(lg, ref, tok, msk, 0.1, inplace=True)
    dl = oo.dlogits.view(B * T, V)
    return torch.matmul(dl, Wh), torch.matmul(dl.t(), hid.view(B * T, d))


for _ in range(2):
    odpo.lmhead_dpo_step(hid, Wh, ref, tok, msk, 0.1)
    unfused()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("chunked")
odpo.lmhead_dpo_step(hid, Wh, ref, tok, msk, 0.1)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
torch.cuda.nvtx.range_push("unfused")
unfused()
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
