"""Factored gradient: the row engine (schedule auto) vs the cluster-split kernel (schedule
split), side by side in one process.  argv: configs.  One JSON line per (config, schedule):
median ms of 9 calls with a 256 MiB L2 flush before each, frac of 1R+1W vs the measured peak."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2410_18252_b200 as odpo  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1].endswith(".so"):
    odpo.LIB_PATH = os.path.abspath(sys.argv.pop(1))
CFG = {"pythia": (256, 53, 50304), "rho": (128, 512, 32000), "llama": (64, 1024, 128256),
       "tiny": (4, 53, 50304)}
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
dev = torch.device("cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for name in sys.argv[1:]:
    P, T, V = CFG[name]
    B = 2 * P
    tok = torch.from_numpy(synth.tokens_rows(0, np.arange(B * T), V).reshape(B, T)).to(dev)
    mask = torch.ones((B, T), dtype=torch.uint8, device=dev)
    x = torch.empty((B, T, V), dtype=torch.bfloat16, device=dev)
    synth.fill_logits_device(x, 0, tokens=tok, peak=14.0)
    ref = odpo.seq_logprobs(x, tok, mask) + torch.linspace(-8, 8, B, device=dev)
    G = torch.empty_like(x)
    for rep in range(2):
        for sched, eng in (("auto", -1), ("split", -1), ("split", 2)):
            times = []
            for i in range(11):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                try:
                    out = odpo.online_dpo_loss_fwd_bwd_unscaled(x, ref, tok, mask, 0.03, G=G,
                                                                schedule=sched, engine=eng)
                except odpo.OdpoError:
                    break   # split: experimental build only
                b.record()
                torch.cuda.synchronize()
                if i >= 2:
                    times.append(a.elapsed_time(b))
            if not times:
                continue
            ms = float(np.median(times))
            print(json.dumps({"config": name, "schedule": sched + ("_tma" if eng == 2 else ""), "ms": ms, "min_ms": min(times),
                              "frac": 2.0 * B * T * V * 2 / (ms / 1e3) / 1e9 / peak,
                              "loss": out.stats[1].item(), "status": int(out.status.item())}),
                  flush=True)
    del x, G, out
    torch.cuda.empty_cache()
