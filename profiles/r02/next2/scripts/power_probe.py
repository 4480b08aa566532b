"""Sustained-loop SM clock / power / time per call of the LLaMA- and Pythia-head forward: cuBLAS's
bf16 GEMM (logits out) vs the library's LM-head forward (tcgen05 GEMM + online-LSE epilogue,
logits never written).  nvidia-smi samples every 50 ms in a side process; one JSON line per
(shape, kernel) with the medians over the window."""
import json
import os
import subprocess
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(
    os.path.abspath(__file__)))))))
import paper_2410_18252_b200 as odpo  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1].endswith(".so"):
    odpo.LIB_PATH = os.path.abspath(sys.argv[1])
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=timestamp,clocks.sm,power.draw",
                        "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)
marks = []
for name, (B, T, d, V) in {"pythia": (512, 53, 2560, 50304), "llama": (128, 1024, 4096, 128256)}.items():
    g = torch.Generator(device="cuda").manual_seed(0)
    hid = (torch.randint(-32, 32, (B, T, d), device="cuda", generator=g).float() / 32).to(torch.bfloat16)
    W = (torch.randint(-32, 32, (V, d), device="cuda", generator=g).float() / 256).to(torch.bfloat16)
    tok = torch.randint(0, V, (B, T), device="cuda", generator=g, dtype=torch.int32)
    mask = torch.ones((B, T), dtype=torch.uint8, device="cuda")
    for kname, fn in (("cublas_gemm", lambda: torch.matmul(hid.view(B * T, d), W.t())),
                      ("odpo_lmhead_fwd", lambda: odpo.lmhead_seq_logprobs(hid, W, tok, mask))):
        fn()
        torch.cuda.synchronize()
        time.sleep(1.0)
        t0 = time.time()
        n = 0
        while time.time() - t0 < 4.0:
            fn()
            n += 1
            if n % 4 == 0:
                torch.cuda.synchronize()
        torch.cuda.synchronize()
        t1 = time.time()
        marks.append((name, kname, t0 + 1.0, t1, (t1 - t0) * 1e3 / n))
    del hid, W
    torch.cuda.empty_cache()
time.sleep(0.3)
smi.terminate()
out = smi.communicate()[0]
samples = []
for line in out.strip().splitlines():
    try:
        ts, clk, pw = [x.strip() for x in line.split(",")]
        t = time.mktime(time.strptime(ts.split(".")[0], "%Y/%m/%d %H:%M:%S")) + float("0." + ts.split(".")[1])
        samples.append((t, float(clk), float(pw)))
    except Exception:
        pass
for name, kname, a, b, ms in marks:
    s = sorted((c, p) for t, c, p in samples if a <= t <= b)
    clk = sorted(c for c, _ in s)
    pw = sorted(p for _, p in s)
    print(json.dumps({"shape": name, "kernel": kname, "ms_per_call": ms,
                      "sm_mhz_median": clk[len(clk) // 2] if clk else None,
                      "power_w_median": pw[len(pw) // 2] if pw else None, "samples": len(s)}), flush=True)
