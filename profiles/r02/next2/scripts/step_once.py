"""One chunked NEXT-2 learner step (LLaMA head) and one unfused cuBLAS step after a warm-up,
for an ncu metrics capture of every GEMM's DRAM / L2 traffic."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(
    os.path.abspath(__file__)))))))
import paper_2410_18252_b200 as odpo  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1].endswith(".so"):
    odpo.LIB_PATH = os.path.abspath(sys.argv[1])
B, T, d, V = 32, 1024, 4096, 128256     # 16 pairs: 32768 rows (one chunk of the step)
g = torch.Generator(device="cuda").manual_seed(0)
hid = (torch.randint(-32, 32, (B, T, d), device="cuda", generator=g).float() / 32).to(torch.bfloat16)
W = (torch.randint(-32, 32, (V, d), device="cuda", generator=g).float() / 256).to(torch.bfloat16)
tok = torch.randint(0, V, (B, T), device="cuda", generator=g, dtype=torch.int32)
msk = torch.ones((B, T), dtype=torch.uint8, device="cuda")
ref = torch.full((B,), -4.0 * T, device="cuda")


def unfused():
    lg = torch.matmul(hid.view(B * T, d), W.t()).view(B, T, V)
    oo = odpo.online_dpo_loss_fwd_bwd(lg, ref, tok, msk, 0.1, inplace=True)
    dl = oo.dlogits.view(B * T, V)
    return torch.matmul(dl, W), torch.matmul(dl.t(), hid.view(B * T, d))


for _ in range(2):
    odpo.lmhead_dpo_step(hid, W, ref, tok, msk, 0.1)
    unfused()
torch.cuda.synchronize()
odpo.lmhead_dpo_step(hid, W, ref, tok, msk, 0.1)
unfused()
torch.cuda.synchronize()
print("ok")
