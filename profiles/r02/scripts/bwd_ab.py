"""A/B of the scaled loss call's row backward (TWO_PASS = AUTO): this build vs variant libraries
(build_variants/libodpo_bwd<cfg>.so, -DODPO_BWD_CFG=cfg).  argv: lib ("main" or a path), then
configs.  Prints one JSON line per config: median loss-call ms over 9 calls with a 256 MiB L2
flush before each, the frac of 1R+1W bytes vs the measured peak, and a hash of dlogits (equal
hashes across libraries = bit-identical outputs)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2410_18252_b200 as odpo  # noqa: E402

PV = -1
if "--pv" in sys.argv:   # exp2_split variant (odpo_launch_opts.exp2_split)
    i = sys.argv.index("--pv")
    PV = int(sys.argv[i + 1])
    del sys.argv[i:i + 2]
lib = sys.argv[1]
if lib != "main":
    odpo.LIB_PATH = os.path.abspath(lib)
CFG = {"pythia": (256, 53, 50304), "rho": (128, 512, 32000), "llama": (64, 1024, 128256),
       "tiny": (4, 53, 50304)}
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
dev = torch.device("cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for name in sys.argv[2:]:
    P, T, V = CFG[name]
    B = 2 * P
    tok = torch.from_numpy(synth.tokens_rows(0, np.arange(B * T), V).reshape(B, T)).to(dev)
    mask = torch.ones((B, T), dtype=torch.uint8, device=dev)
    x = torch.empty((B, T, V), dtype=torch.bfloat16, device=dev)
    synth.fill_logits_device(x, 0, tokens=tok, peak=14.0)
    ref = odpo.seq_logprobs(x, tok, mask) + torch.linspace(-8, 8, B, device=dev)
    dl = torch.empty_like(x)
    times = []
    for i in range(11):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = odpo.online_dpo_loss_fwd_bwd(x, ref, tok, mask, 0.03, dlogits=dl, exp2_split=PV)
        b.record()
        torch.cuda.synchronize()
        if i >= 2:
            times.append(a.elapsed_time(b))
    ms = float(np.median(times))
    w = dl.view(torch.int16).view(-1)
    h = int((w[::7].to(torch.int64) * 2654435761 % 1000003).sum().item())
    alg = 2.0 * B * T * V * 2
    print(json.dumps({"lib": lib, "pv": PV, "config": name, "ms": ms, "min_ms": min(times),
                      "frac": alg / (ms / 1e3) / 1e9 / peak, "hash": h,
                      "loss": out.stats[1].item()}), flush=True)
    del x, dl, out
    torch.cuda.empty_cache()
