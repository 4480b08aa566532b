# SM clock and power while the fused LM-head kernel and cuBLAS run the LLaMA head (sustained)
mkdir -p gpurun_out
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv -lms 50 > gpurun_out/lmh_clocks.csv &
SMI=$!
python - > gpurun_out/lmh_clock_probe.log 2>&1 <<'PY'
import time, torch, sys
sys.path.insert(0, ".")
import paper_2410_18252_b200 as odpo
B, T, d, V = 128, 1024, 4096, 128256
g = torch.Generator(device="cuda").manual_seed(0)
hid = (torch.randint(-32, 32, (B, T, d), device="cuda", generator=g).float() / 32).to(torch.bfloat16)
W = (torch.randint(-32, 32, (V, d), device="cuda", generator=g).float() / 256).to(torch.bfloat16)
tok = torch.randint(0, V, (B, T), device="cuda", generator=g, dtype=torch.int32)
mask = torch.ones((B, T), dtype=torch.uint8, device="cuda")
def run(name, fn, n=20):
    torch.cuda.synchronize(); t0 = time.time()
    print(name, "start", t0, flush=True)
    for _ in range(n): fn()
    torch.cuda.synchronize(); t1 = time.time()
    print(name, "end", t1, "ms/call", (t1 - t0) * 1e3 / n, flush=True)
run("fused", lambda: odpo.lmhead_seq_logprobs(hid, W, tok, mask))
time.sleep(1.0)
run("cublas", lambda: torch.matmul(hid.view(B * T, d), W.t()))
PY
kill $SMI
