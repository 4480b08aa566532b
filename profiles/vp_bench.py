#!/usr/bin/env python
"""NEXT-4 measurement on one GPU: the per-rank kernels of a W-way vocabulary-parallel step
(partials over the shard, merge + pair reduce + shard backward), timed shard by shard with CUDA
events; under torchrun (ranks sharing or owning GPUs) the full vp_loss_step with its
all-gather.  Prints one JSON line."""
import argparse
import json
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
    ap.add_argument("--config", default="llama")
    ap.add_argument("--W", type=int, default=8)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--put", action="store_true",
                    help="the in-kernel exchange (odpo_vp_row_partials_put + the waiting merge), "
                         "the W ranks' buffers emulated on this GPU")
    ap.add_argument("--lib", default=None, help="a variant build of libodpo.so (A/B)")
    a = ap.parse_args()
    if a.lib:
        odpo.LIB_PATH = os.path.abspath(a.lib)
    w = CONFIGS[a.config]
    B, T, V = 2 * w.P, w.T, w.V
    dev = torch.device("cuda:0")
    tok = torch.from_numpy(synth.tokens_rows(0, np.arange(B * T), V).reshape(B, T)).to(dev)
    mask = torch.ones((B, T), dtype=torch.uint8, device=dev)
    Vs = -(-V // a.W)
    Vs = -(-Vs // 8) * 8
    v0 = 0  # time shard 0 (all shards have the same size but the last)
    x = torch.empty((B, T, Vs), dtype=torch.bfloat16, device=dev)
    synth.fill_logits_device(x, 0, tokens=torch.clamp(tok, max=Vs - 1))
    dl = torch.empty_like(x)
    ref = torch.full((B,), -0.08 * T, device=dev)
    parts = odpo.vp_row_partials(x, v0, V, tok, mask)
    parts_all = torch.stack([parts] * a.W)
    ex = odpo.VPExchange.emulate(a.W, B * T) if a.put else None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    tp, tl = [], []
    for i in range(a.reps + 2):
        flush.zero_()
        if ex is not None:   # the other ranks' puts of this epoch land first (untimed)
            for r in range(1, a.W):
                odpo.vp_row_partials_put(x, v0, V, tok, mask, ex[r], i + 1)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        if ex is None:
            odpo.vp_row_partials(x, v0, V, tok, mask)
        else:
            odpo.vp_row_partials_put(x, v0, V, tok, mask, ex[0], i + 1)
        e[1].record()
        if ex is None:
            odpo.vp_loss_fwd_bwd(parts_all, x, v0, V, ref, tok, mask, w.beta, dlogits=dl)
        else:
            odpo.vp_loss_fwd_bwd(ex[0].parts(i + 1), x, v0, V, ref, tok, mask, w.beta, dlogits=dl,
                                 flags=ex[0].flags(), epoch=i + 1)
        e[2].record()
        torch.cuda.synchronize()
        if i >= 2:
            tp.append(e[0].elapsed_time(e[1]))
            tl.append(e[1].elapsed_time(e[2]))
    shard_bytes = B * T * Vs * 2
    t = np.mean(tp) + np.mean(tl)
    alg = 2 * shard_bytes
    print(json.dumps({"what": "vocab-parallel per-rank kernels (one shard, timed on one GPU)",
                      "exchange": "in-kernel put + flag wait" if a.put else "caller all-gather",
                      "config": a.config, "W": a.W, "V_shard": Vs,
                      "partials_ms": float(np.mean(tp)), "loss_bwd_ms": float(np.mean(tl)),
                      "rank_ms": float(t), "alg_GBs": alg / t / 1e6,
                      "frac_1R1W": alg / t / 1e6 / 6546.9,
                      "dram_traffic_model": "2R+1W of the shard (forward and backward reads)"}))


if __name__ == "__main__":
    main()
