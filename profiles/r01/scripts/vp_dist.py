#!/usr/bin/env python
"""torchrun check of vp_loss_step: each rank owns one vocabulary shard; the result must equal
the single-process unsharded loss (rank 0 prints it)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402
import paper_2410_18252_b200 as odpo  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    dist.init_process_group(os.environ.get("ODPO_DIST_BACKEND", "nccl"))
    P, T, V = 8, 17, 32000
    B = 2 * P
    tok = torch.from_numpy(synth.tokens_rows(0, np.arange(B * T), V).reshape(B, T)).to(dev)
    mask = torch.ones((B, T), dtype=torch.uint8, device=dev)
    x = torch.empty((B, T, V), dtype=torch.bfloat16, device=dev)
    synth.fill_logits_device(x, 0, tokens=tok)
    ref = torch.full((B,), -1.5, device=dev)
    cuts = [((V * r) // world) // 8 * 8 for r in range(world)] + [V]
    a, e = cuts[rank], cuts[rank + 1]
    out = odpo.vp_loss_step(x[:, :, a:e], a, V, ref, tok, mask, 0.1)
    full = odpo.online_dpo_loss_fwd_bwd(x, ref, tok, mask, 0.1)
    torch.cuda.synchronize()
    rel = float((out.stats[1] - full.stats[1]).abs() / full.stats[1].abs())
    dmax = float((out.dlogits.float() - full.dlogits[:, :, a:e].float()).abs().max())
    ok = rel < 1e-5 and dmax < 1e-6 and int(out.status.item()) == 0
    flag = torch.tensor([1 if ok else 0], device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(f"vp_dist world={world} loss={out.stats[1].item():.6f} full={full.stats[1].item():.6f} "
              f"rel={rel:.2e} max|ddl|={dmax:.2e} ok={bool(flag.item())}")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
