"""NEXT-4: vocabulary-parallel loss, W shards of the vocabulary emulated on one GPU (the
all-gather of the row partials is a torch.stack here; NCCL all_gather_into_tensor across
ranks in vp_loss_step).  Compared with the unsharded oracle."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_helpers import NCPU, Batch, check_dlogits, check_seq, check_stats, coef_from_oracle, to_f64

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def odpo():
    import paper_2410_18252_b200 as m
    m._L()
    return m


def shard_bounds(V, W, align):
    """W contiguous column ranges, inner boundaries on multiples of `align` elements (the
    16-byte alignment of every shard base)."""
    cuts = [0] + [((V * w) // W) // align * align for w in range(1, W)] + [V]
    return list(zip(cuts[:-1], cuts[1:]))


@pytest.mark.parametrize("W", [1, 3, 8])
@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_vp_parity(odpo, W, dt):
    P, T, V = 3, 9, 12345 if dt == "f32" else 32000
    b = Batch(P, T, V, dt, seed=7, mask_kind="prefix", lbar=5, extra_seqs=1)
    ref = (synth.rewards_for(7, b.B, 1).reshape(-1) - 20.0).astype(np.float32)
    d_ref = torch.from_numpy(ref).cuda()
    align = 8 if dt == "bf16" else 4
    bounds = shard_bounds(V, W, align)
    parts = [odpo.vp_row_partials(b.d_logits[:, :, a:e], a, V, b.d_tokens, b.d_mask)
             for a, e in bounds]
    parts_all = torch.stack(parts)
    dl = b.new_out()
    outs = [odpo.vp_loss_fwd_bwd(parts_all, b.d_logits[:, :, a:e], a, V, d_ref, b.d_tokens,
                                 b.d_mask, 0.1, pair_rows=b.d_pair_rows, p_global=P + 1,
                                 dlogits=dl[:, :, a:e]) for a, e in bounds]
    torch.cuda.synchronize()
    o = oracle.online_dpo_loss_fwd_bwd(b.h_logits, ref, b.tokens, b.mask, 0.1,
                                       pair_rows=b.pair_rows, p_global=P + 1, want_dlogits=True,
                                       n_threads=NCPU)
    live = b.pair_rows.reshape(-1)
    for out in outs:   # every rank of the vocabulary group holds the same global results
        assert torch.equal(out.seq_logp[torch.from_numpy(live).cuda()],
                           outs[0].seq_logp[torch.from_numpy(live).cuda()])
        assert torch.equal(out.stats[:10], outs[0].stats[:10])
        assert int(out.status.item()) == 0
    check_seq(outs[0].seq_logp.cpu().numpy()[live], o["seq_logp"][live], dt)
    check_stats(outs[0].stats.cpu().numpy(), o, dt, 0.1, ref, b.pair_rows, Pg=P + 1)
    coef = coef_from_oracle(o, P, P + 1, 0.1, 1.0, b.pair_rows, b.B)
    check_dlogits(to_f64(dl), o["dlogits"], coef[:, None, None], dt)


def test_vp_token_ownership_flags(odpo):
    """A token outside [0, V_total) is flagged; every in-range token has exactly one owner."""
    b = Batch(2, 5, 4096, "bf16", seed=8, host=False)
    parts = [odpo.vp_row_partials(b.d_logits[:, :, a:e], a, 4096, b.d_tokens, b.d_mask)
             for a, e in shard_bounds(4096, 4, 8)]
    owners = torch.stack(parts)[:, :, 3].sum(0)
    assert torch.all(owners[b.d_mask.reshape(-1).bool()] == 1)
    tok = b.d_tokens.clone()
    tok[0, 0] = 4096
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    odpo.vp_row_partials(b.d_logits[:, :, 0:2048], 0, 4096, tok, b.d_mask, status=st)
    torch.cuda.synchronize()
    assert int(st.item()) & odpo.FLAGS["TOKEN_RANGE"]
