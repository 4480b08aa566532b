#!/usr/bin/env python
"""Run every libodpo entry point once on small shapes (the tiny config's T and V) for
compute-sanitizer: memcheck / racecheck / synccheck / initcheck."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2410_18252_b200 as odpo  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    P, T, V = 4, 53, 50304
    B = 2 * P
    for dtype in (torch.float32, torch.bfloat16):
        tok = torch.from_numpy(synth.tokens_rows(0, np.arange(B * T), V).reshape(B, T)).to(dev)
        mask = torch.from_numpy(synth.mask_for(0, np.arange(B), T, "prefix", 26)).to(dev)
        x = torch.empty((B, T, V), dtype=dtype, device=dev)
        synth.fill_logits_device(x, 0, tokens=tok)
        rew = torch.from_numpy(synth.rewards_for(0, P, 2)).to(dev)
        sel = odpo.pair_select(rew)
        ref = odpo.seq_logprobs(x, tok, mask)
        for sched in ("fused", "two_pass", "wave"):
            odpo.online_dpo_loss_fwd_bwd(x, ref, tok, mask, 0.05, pair_rows=sel.pair_rows,
                                         schedule=sched)
        odpo.online_dpo_loss_fwd_bwd_unscaled(x, ref, tok, mask, 0.05, pair_rows=sel.pair_rows)
        odpo.online_dpo_loss_fwd_bwd_unscaled(x, ref, tok, mask, 0.05, engine=1)
        for kind in ("rloo", "copg", "prox_rloo", "sft"):
            odpo.pg_loss_fwd_bwd(x, tok, mask, kind, rew.reshape(-1), ref, 0.2,
                                 pair_rows=sel.pair_rows)
        rew4 = torch.from_numpy(synth.rewards_for(0, 2, 4)).to(dev)
        sel4 = odpo.pair_select(rew4)
        odpo.gather_pairs(sel4.pair_rows, tok, mask, ref)
        odpo.seq_ppl(x, tok, mask)
        # NEXT-4: two vocabulary shards, partials exchanged in the kernels (emulated peers)
        h = V // 2 // 8 * 8
        ex = odpo.VPExchange.emulate(2, B * T)
        for r, (a, e) in enumerate(((0, h), (h, V))):
            odpo.vp_row_partials_put(x[:, :, a:e], a, V, tok, mask, ex[r], 1)
        for r, (a, e) in enumerate(((0, h), (h, V))):
            odpo.vp_loss_fwd_bwd(ex[r].parts(1), x[:, :, a:e], a, V, ref, tok, mask, 0.05,
                                 pair_rows=sel.pair_rows, flags=ex[r].flags(), epoch=1)
        torch.cuda.synchronize()
    # NEXT-2: LM-head forward, loss, and the tcgen05 backward GEMMs on a small head
    d, Vh = 256, 3001
    hid, W = synth.lmhead_inputs(0, np.arange(B * T), d, Vh)
    hd = torch.from_numpy(hid.reshape(B, T, d).astype(np.float32)).to(dev).to(torch.bfloat16)
    wd = torch.from_numpy(W.astype(np.float32)).to(dev).to(torch.bfloat16)
    tk = torch.from_numpy(synth.tokens_rows(0, np.arange(B * T), Vh).reshape(B, T)).to(dev)
    o = odpo.lmhead_online_dpo_loss_fwd(hd, wd, torch.full((B,), -30.0, device=dev), tk, mask, 0.05)
    odpo.lmhead_grad(hd, wd, tk, o.row_lse, o.row_scale, chunk_rows=256)
    torch.cuda.synchronize()
    print("sanitize run ok")


if __name__ == "__main__":
    main()
