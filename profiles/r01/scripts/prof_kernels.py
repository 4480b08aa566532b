#!/usr/bin/env python
"""Launch each hot-path kernel variant a few times on one workload, for ncu captures.

    python profiles/prof_kernels.py --config pythia --variants fused:0,fused:3,two_pass:0,seq
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2410_18252_b200 as odpo  # noqa: E402
from synth.configs import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="pythia")
    ap.add_argument("--variants", default="fused:-1,seq")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--lag", type=int, default=0)
    a = ap.parse_args()
    w = CONFIGS[a.config]
    dev = torch.device("cuda:0")
    B, T, V = 2 * w.P, w.T, w.V
    tdt = torch.bfloat16 if w.dtype == "bf16" else torch.float32
    rows = np.arange(B * T)
    tokens = torch.from_numpy(synth.tokens_rows(0, rows, V).reshape(B, T)).to(dev)
    mask = torch.from_numpy(synth.mask_for(0, np.arange(B), T, "dense")).to(dev)
    logits = torch.empty((B, T, V), dtype=tdt, device=dev)
    synth.fill_logits_device(logits, 0, tokens=tokens)
    dl = torch.empty_like(logits)
    ref = torch.full((B,), -0.08 * T, device=dev)
    for v in a.variants.split(","):
        for _ in range(a.reps):
            if v == "seq":
                odpo.seq_logprobs(logits, tokens, mask)
            elif v == "unsc":
                odpo.online_dpo_loss_fwd_bwd_unscaled(logits, ref, tokens, mask, w.beta, G=dl)
            else:
                parts = v.split(":")
                sched, split = parts[0], int(parts[1]) if len(parts) > 1 else -1
                lag = int(parts[2]) if len(parts) > 2 else a.lag
                odpo.online_dpo_loss_fwd_bwd(logits, ref, tokens, mask, w.beta, dlogits=dl,
                                             schedule=sched, exp2_split=split, lag_pairs=lag)
        torch.cuda.synchronize()
    print("done")


if __name__ == "__main__":
    main()
