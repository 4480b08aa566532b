"""One LLaMA-head forward of each kind (cuBLAS GEMM, the library's LM-head forward) after a
warm-up, for an ncu metrics capture of their DRAM / L2 traffic."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(
    os.path.abspath(__file__)))))))
import paper_2410_18252_b200 as odpo  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1].endswith(".so"):
    odpo.LIB_PATH = os.path.abspath(sys.argv[1])
B, T, d, V = 128, 1024, 4096, 128256
g = torch.Generator(device="cuda").manual_seed(0)
hid = (torch.randint(-32, 32, (B, T, d), device="cuda", generator=g).float() / 32).to(torch.bfloat16)
W = (torch.randint(-32, 32, (V, d), device="cuda", generator=g).float() / 256).to(torch.bfloat16)
tok = torch.randint(0, V, (B, T), device="cuda", generator=g, dtype=torch.int32)
mask = torch.ones((B, T), dtype=torch.uint8, device="cuda")
for _ in range(2):
    torch.matmul(hid.view(B * T, d), W.t())
    odpo.lmhead_seq_logprobs(hid, W, tok, mask)
torch.cuda.synchronize()
torch.matmul(hid.view(B * T, d), W.t())
odpo.lmhead_seq_logprobs(hid, W, tok, mask)
torch.cuda.synchronize()
print("ok")
