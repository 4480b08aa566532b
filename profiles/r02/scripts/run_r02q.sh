timeout 900 python -m pytest tests/test_lmhead.py tests/test_abi.py -q -x --timeout 600 2>&1 | tail -3
timeout 600 python profiles/r02/lmhead_grad_bench.py --quick 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_gemm|k_engine|k_prep|k_stats" --csv --log-file /tmp/cl.csv python -c "
import sys, torch
sys.path.insert(0, '.')
import paper_2410_18252_b200 as odpo
B, T, d, V = 512, 53, 2560, 50304
g = torch.Generator(device='cuda').manual_seed(0)
hid = (torch.randint(-32, 32, (B, T, d), device='cuda', generator=g).float() / 32).to(torch.bfloat16)
Wh = (torch.randint(-32, 32, (V, d), device='cuda', generator=g).float() / 256).to(torch.bfloat16)
tok = torch.randint(0, V, (B, T), device='cuda', generator=g, dtype=torch.int32)
msk = torch.ones((B, T), dtype=torch.uint8, device='cuda')
ref = torch.full((B,), -4.0 * T, device='cuda')
for _ in range(2): odpo.lmhead_dpo_step(hid, Wh, ref, tok, msk, 0.1)
torch.cuda.synchronize()
" > /dev/null 2>&1
python profiles/summarize_ncu.py r02q_chunked pythia chunked /tmp/cl.csv 2>&1 | grep "k_"
