"""GPU checks of the call contract (include/odpo.h "General conventions"; VERDICT r1 weak #7,
ADVICE r1): calls on different streams do not share scratch, the binding rejects mis-shaped
outputs before any launch, a masked row with huge logits cannot poison the LM-head gradient,
and the KL proxy (odpo_seq_ppl) matches the oracle."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_helpers import NCPU, TOL_SEQ, Batch, check_seq

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def odpo():
    import paper_2410_18252_b200 as m
    m._L()
    return m


def test_concurrent_streams_match_serial(odpo):
    """Two loss calls (different batches and shapes) in flight at once on two streams give the
    same bits as each run alone: every stream has its own workspace (k_prep counters, ring
    state) and AUTO never selects a schedule that needs co-residency."""
    a = Batch(64, 53, 50304, "bf16", seed=40, host=False)
    b = Batch(9, 17, 32000, "bf16", seed=41, mask_kind="prefix", lbar=9, host=False)
    ref_a = torch.full((a.B,), -4.0, device="cuda")
    ref_b = torch.full((b.B,), -6.0, device="cuda")
    serial_a = odpo.online_dpo_loss_fwd_bwd(a.d_logits, ref_a, a.d_tokens, a.d_mask, 0.1)
    serial_b = odpo.online_dpo_loss_fwd_bwd(b.d_logits, ref_b, b.d_tokens, b.d_mask, 0.05)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for _ in range(4):
        with torch.cuda.stream(s1):
            oa = odpo.online_dpo_loss_fwd_bwd(a.d_logits, ref_a, a.d_tokens, a.d_mask, 0.1)
        with torch.cuda.stream(s2):
            ob = odpo.online_dpo_loss_fwd_bwd(b.d_logits, ref_b, b.d_tokens, b.d_mask, 0.05)
        outs.append((oa, ob))
    torch.cuda.synchronize()
    for oa, ob in outs:
        assert torch.equal(oa.dlogits, serial_a.dlogits) and torch.equal(oa.stats, serial_a.stats)
        assert torch.equal(ob.dlogits, serial_b.dlogits) and torch.equal(ob.stats, serial_b.stats)
        assert int(oa.status.item()) == 0 and int(ob.status.item()) == 0


def test_binding_rejects_misshaped_buffers(odpo):
    b = Batch(2, 5, 1000, "bf16", seed=42, host=False)
    ref = torch.zeros(b.B, device="cuda")
    bad_dl = torch.empty((b.B, b.T - 1, b.V), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(odpo.OdpoError):
        odpo.online_dpo_loss_fwd_bwd(b.d_logits, ref, b.d_tokens, b.d_mask, 0.1, dlogits=bad_dl)
    with pytest.raises(odpo.OdpoError):
        odpo.online_dpo_loss_fwd_bwd(b.d_logits, ref, b.d_tokens, b.d_mask, 0.1,
                                     stats=torch.zeros(16, dtype=torch.float32, device="cuda"))
    with pytest.raises(odpo.OdpoError):
        odpo.online_dpo_loss_fwd_bwd(b.d_logits, ref, b.d_tokens, b.d_mask, 0.1,
                                     stats=torch.zeros(4, dtype=torch.float64, device="cuda"))
    with pytest.raises(odpo.OdpoError):
        odpo.online_dpo_loss_fwd_bwd(b.d_logits, ref, b.d_tokens, b.d_mask, 0.1,
                                     status=torch.zeros(1, dtype=torch.float32, device="cuda"))
    with pytest.raises(odpo.OdpoError):
        odpo.online_dpo_loss_fwd_bwd(b.d_logits, ref[:-1], b.d_tokens, b.d_mask, 0.1)
    with pytest.raises(odpo.OdpoError):
        odpo.online_dpo_loss_fwd_bwd(b.d_logits, ref, b.d_tokens[:, :-1], b.d_mask, 0.1)
    with pytest.raises(odpo.OdpoError):
        odpo.online_dpo_loss_fwd_bwd_unscaled(
            b.d_logits, ref, b.d_tokens, b.d_mask, 0.1,
            G=torch.empty((b.B, b.T, b.V + 8), dtype=torch.bfloat16, device="cuda"))
    with pytest.raises(odpo.OdpoError):
        odpo.pg_loss_fwd_bwd(b.d_logits, b.d_tokens, b.d_mask, "rloo", ref[:2])
    with pytest.raises(odpo.OdpoError):
        odpo.online_dpo_loss_fwd_bwd(b.d_logits, ref, b.d_tokens, b.d_mask, 0.1,
                                     pair_rows=torch.zeros((2, 3), dtype=torch.int32, device="cuda"))


def test_lmhead_grad_masked_rows_with_huge_logits_stay_finite(odpo):
    """a masked row (row_scale 0) whose logits exceed exp's range must produce exact
    zeros in G, hence finite dhidden / dweight."""
    B, T, d, V = 2, 128, 64, 512
    rows = np.arange(B * T)
    h, w = synth.lmhead_inputs(3, rows, d, V)
    h = h.reshape(B, T, d)
    h[1, :, :] = 30.0          # masked sequence: logits ~ 30 * 64 * |w| >> 88
    w = np.abs(w) + 0.5
    tok = synth.tokens_rows(3, rows, V).reshape(B, T).astype(np.int32)
    mask = np.ones((B, T), np.uint8)
    mask[1] = 0
    hd = torch.from_numpy(h.astype(np.float32)).to(torch.bfloat16).cuda()
    wd = torch.from_numpy(w.astype(np.float32)).to(torch.bfloat16).cuda()
    tk, mk = torch.from_numpy(tok).cuda(), torch.from_numpy(mask).cuda()
    _, _, lse, _ = odpo.lmhead_seq_logprobs(hd, wd, tk, mk)
    row_scale = torch.ones((B, T), device="cuda") * 1e-3
    row_scale[1] = 0.0
    dh, dw = odpo.lmhead_grad(hd, wd, tk, lse, row_scale)
    torch.cuda.synchronize()
    assert torch.isfinite(dh).all() and torch.isfinite(dw).all()
    assert torch.count_nonzero(dh[1]).item() == 0


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_seq_ppl_parity(odpo, dtype):
    """KL proxy: per-completion perplexity exp(-S_b / n_b) and its fixed-order sums against
    the oracle; an empty completion is flagged and gets 1."""
    P, T, V = 5, 19, 50304
    b = Batch(P, T, V, dtype, seed=43, mask_kind="prefix", lbar=9)
    mask = b.mask.copy()
    mask[3] = 0
    d_mask = torch.from_numpy(mask).cuda()
    ppl, ps, seq, status = odpo.seq_ppl(b.d_logits, b.d_tokens, d_mask)
    torch.cuda.synchronize()
    o = oracle.seq_ppl(b.h_logits, b.tokens, mask, n_threads=NCPU)
    assert int(status.item()) & odpo.FLAGS["EMPTY_SEQ"] and o["status"] & oracle.FLAG_EMPTY_SEQ
    check_seq(seq.cpu().numpy(), o["seq_logp"], dtype)
    n = mask.sum(1).astype(np.float64)
    tol = TOL_SEQ[dtype]
    # |d ppl| / ppl = |dS| / n with |dS| <= tol max(|S|, 1)  (+ the fp32 rounding of ppl)
    bound = (tol * np.maximum(np.abs(o["seq_logp"]), 1.0) / np.maximum(n, 1) + 2.0 ** -23) * o["ppl"]
    assert np.all(np.abs(ppl.cpu().double().numpy() - o["ppl"]) <= bound)
    assert ppl[3].item() == 1.0
    g = ps.cpu().numpy()
    assert g[0] == o["ppl_stats"][0] and g[3] == o["ppl_stats"][3]
    assert abs(g[1] - o["ppl_stats"][1]) <= bound.sum()
    assert abs(g[2] - o["ppl_stats"][2]) <= tol * np.maximum(np.abs(o["seq_logp"]), 1.0).sum()


def test_seq_ppl_uniform_rows_is_V(odpo):
    """Uniform rows: every token has probability 1/V, so PPL = V exactly (closed form)."""
    B, T, V = 3, 7, 32000
    x = torch.full((B, T, V), 0.375, dtype=torch.bfloat16, device="cuda")
    tok = torch.from_numpy(synth.tokens_rows(1, np.arange(B * T), V).reshape(B, T)).cuda()
    mask = torch.ones((B, T), dtype=torch.uint8, device="cuda")
    ppl, ps, _, _ = odpo.seq_ppl(x, tok, mask)
    torch.cuda.synchronize()
    assert torch.all(torch.abs(ppl.double() - V) <= 2e-3 * V / T)
    assert abs(math.exp(-ps[2].item() / ps[3].item()) - V) <= 2e-3 * V
