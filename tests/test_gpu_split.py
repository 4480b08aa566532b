"""GPU-vs-oracle parity of the cluster-split factored gradient (schedule "split",
ODPO_SCHED_SPLIT: each row over a thread-block cluster of up to 8 CTAs, one register-held
vocabulary piece per CTA, the partials merged through distributed shared memory).  Same
contract as the engine's factored call (tests/test_gpu_unscaled.py): G = mask (softmax -
onehot), row_scale = coef_b mask, against oracle.online_dpo_loss_fwd_bwd(..., unscaled=True)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_helpers import NCPU, Batch, alloc_rows, check_dlogits, check_seq, check_stats, to_f64
from test_gpu_unscaled import check_row_scale

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def odpo():
    import paper_2410_18252_b200 as m
    m._L()
    return m


ENGINE = -1   # the register-held pieces; test_split_tma_* rerun the cases with engine=2


def split(odpo, b, ref, beta, Pg=None, **kw):
    if not kw.get("inplace"):
        kw.setdefault("G", b.new_out())
    try:
        out = odpo.online_dpo_loss_fwd_bwd_unscaled(b.d_logits, ref, b.d_tokens, b.d_mask, beta,
                                                    pair_rows=b.d_pair_rows, p_global=Pg,
                                                    inv_temperature=b.invT, schedule="split",
                                                    engine=kw.pop("engine", ENGINE), **kw)
    except odpo.OdpoError as e:
        # SPLIT is compiled only in the experimental build (measured slower than the row
        # engine): run with --odpo-lib build_variants/libodpo_experimental.so
        if "unsupported" in str(e):
            pytest.skip(f"split schedule not in this build: {e}")
        raise
    torch.cuda.synchronize()
    return out


CASES = [
    # (P, T, V, dtype, mask, extra_seqs, invT): 16-byte (V = 4133, 8, 12345 f32) and 32-byte
    # (V = 32000, 50304) rows, 1 / 2 / 4 / 8 CTAs per row, ragged tails, unreferenced sequences
    (3, 5, 4133, "bf16", "prefix", 2, 1.0),
    (3, 5, 4133, "f32", "prefix", 1, 1 / 0.7),
    (2, 9, 8, "bf16", "dense", 1, 1.0),
    (5, 17, 32000, "bf16", "prefix", 0, 1.0),
    (2, 7, 12345, "f32", "dense", 0, 1.0),
    (2, 6, 50304, "bf16", "dense", 1, 1.0),
    (2, 4, 128256, "bf16", "prefix", 0, 2.0),
    (1, 3, 40000, "f32", "dense", 0, 1.0),
    (2, 3, 131069, "bf16", "dense", 0, 1.0),
]


@pytest.mark.parametrize("eng", [-1, 2], ids=["regs", "tma"])
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"P{c[0]}T{c[1]}V{c[2]}{c[3]}{c[4]}x{c[5]}")
def test_split_parity_small(odpo, case, eng):
    P, T, V, dt, mk, extra, invT = case
    b = Batch(P, T, V, dt, seed=3, mask_kind=mk, lbar=max(1, T // 2), extra_seqs=extra, invT=invT)
    ref = (synth.rewards_for(3, b.B, 1).reshape(-1) - 30.0).astype(np.float32)
    beta, Pg = 0.1, P + 2
    d_ref = torch.from_numpy(ref).cuda()
    out = split(odpo, b, d_ref, beta, Pg=Pg, engine=eng)
    assert out.launches == 2
    o = oracle.online_dpo_loss_fwd_bwd(b.h_logits, ref, b.tokens, b.mask, beta,
                                       pair_rows=b.pair_rows, p_global=Pg, inv_temperature=invT,
                                       want_dlogits=True, n_threads=NCPU, unscaled=True)
    live = np.arange(b.B) if b.pair_rows is None else b.pair_rows.reshape(-1)
    check_seq(out.seq_logp.cpu().numpy()[live], o["seq_logp"][live], dt)
    check_dlogits(to_f64(out.dlogits), o["dlogits"], 1.0, dt)
    check_row_scale(out.row_scale.cpu().numpy(), o["row_scale"], dt)
    check_stats(out.stats.cpu().numpy(), o, dt, beta, ref, b.pair_rows, Pg=Pg)
    assert int(out.status.item()) == 0
    if extra:
        unref = np.setdiff1d(np.arange(b.B), live)
        assert torch.count_nonzero(out.dlogits[torch.from_numpy(unref).cuda()]).item() == 0
        assert torch.count_nonzero(out.row_scale[torch.from_numpy(unref).cuda()]).item() == 0


def test_split_inplace_deterministic_and_engine_agreement(odpo):
    P, T, V = 6, 13, 50304
    b = Batch(P, T, V, "bf16", seed=8, mask_kind="prefix", lbar=7, host=False)
    ref = torch.full((b.B,), -10.0, device="cuda")
    a1 = split(odpo, b, ref, 0.1)
    a2 = split(odpo, b, ref, 0.1)
    assert torch.equal(a1.dlogits, a2.dlogits) and torch.equal(a1.row_scale, a2.row_scale)
    assert torch.equal(a1.stats, a2.stats)
    x = alloc_rows(b.B, b.T, b.V, "bf16")
    x.copy_(b.d_logits)
    bi = Batch.__new__(Batch)
    bi.__dict__.update(b.__dict__)
    bi.d_logits = x
    a3 = split(odpo, bi, ref, 0.1, inplace=True)
    assert a3.dlogits.data_ptr() == x.data_ptr()
    assert torch.equal(a3.dlogits, a1.dlogits) and torch.equal(a3.stats, a1.stats)
    # the engine's factored call: the same quantities through another reduction tree
    e = odpo.online_dpo_loss_fwd_bwd_unscaled(b.d_logits, ref, b.d_tokens, b.d_mask, 0.1,
                                              G=b.new_out())
    torch.cuda.synchronize()
    assert torch.allclose(e.seq_logp, a1.seq_logp, rtol=1e-5, atol=1e-4)
    assert torch.allclose(e.row_scale, a1.row_scale, rtol=1e-4, atol=0)
    d = (e.dlogits.float() - a1.dlogits.float()).abs()
    assert float((d - 2.0 ** -7 * e.dlogits.float().abs()).max()) <= 2.0 ** -20


def test_split_best_worst_of_k4(odpo):
    """K = 4 completions per prompt: the 2 unselected ones are unreferenced sequences, zeroed
    by the kernel's zero workers (G = 0, row_scale = 0)."""
    P, K, T, V = 16, 4, 9, 3001
    rewards = synth.rewards_for(6, P, K, kind="verifier")
    eos = synth.has_eos_for(6, P, K)
    sel = odpo.pair_select(torch.from_numpy(rewards).cuda(), torch.from_numpy(eos).cuda(), -1.0)
    o_sel = oracle.pair_select(rewards, eos, -1.0)
    b = Batch(P, T, V, "bf16", seed=6, mask_kind="prefix", lbar=5, extra_seqs=(K - 2) * P)
    b.pair_rows = o_sel["pair_rows"].astype(np.int32)
    b.d_pair_rows = sel.pair_rows
    ref = np.full(b.B, -0.5 * T, np.float32)
    G = b.new_out()
    G.fill_(7.0)   # every entry must be written
    out = split(odpo, b, torch.from_numpy(ref).cuda(), 0.1, G=G)
    o = oracle.online_dpo_loss_fwd_bwd(b.h_logits, ref, b.tokens, b.mask, 0.1,
                                       pair_rows=b.pair_rows, want_dlogits=True, n_threads=NCPU,
                                       unscaled=True)
    check_dlogits(to_f64(out.dlogits), o["dlogits"], 1.0, "bf16")
    check_row_scale(out.row_scale.cpu().numpy(), o["row_scale"], "bf16")


def test_split_poisoned_and_token_range(odpo):
    """Status flags as the engine raises them: a NaN logit, a token outside [0, V)."""
    P, T, V = 2, 3, 5000
    b = Batch(P, T, V, "bf16", seed=1, host=False)
    b.d_logits[0, 1, 17] = float("nan")
    ref = torch.full((b.B,), -10.0, device="cuda")
    out = split(odpo, b, ref, 0.1)
    assert int(out.status.item()) & 2
    tok = b.d_tokens.clone()
    tok[1, 2] = V + 5
    bt = Batch.__new__(Batch)
    bt.__dict__.update(b.__dict__)
    bt.d_tokens = tok
    out = split(odpo, bt, ref, 0.1)
    assert int(out.status.item()) & 1


@pytest.mark.parametrize("eng", [-1, 2], ids=["regs", "tma"])
@pytest.mark.parametrize("name,mask_kind", [("pythia", "dense"), ("rho", "dense"),
                                            ("llama", "prefix")])
def test_split_full_size_sampled(odpo, name, mask_kind, eng):
    """BASELINE.json configs at full size in the bench's launch configuration: sampled rows
    against the oracle, statistics against the engine's factored call."""
    from synth.configs import CONFIGS
    w = CONFIGS[name]
    b = Batch(w.P, w.T, w.V, w.dtype, seed=0, mask_kind=mask_kind, lbar=w.lbar, host=False)
    ref = torch.full((b.B,), -float(w.T) * 0.08, dtype=torch.float32, device="cuda")
    out = split(odpo, b, ref, w.beta, engine=eng)
    assert int(out.status.item()) == 0
    pairs = synth.permutation(1, w.P)[:2]
    seqs = np.stack([2 * pairs, 2 * pairs + 1], 1).reshape(-1)
    h_x = b.host_rows(seqs)
    h_ref = np.full(len(seqs), -float(w.T) * 0.08, np.float32)
    rows = (np.arange(len(seqs))[:, None] * w.T + np.arange(w.T)[None, :])
    take = rows[:, :3].reshape(-1)
    o = oracle.online_dpo_loss_fwd_bwd(h_x, h_ref, b.tokens[seqs], b.mask[seqs], w.beta,
                                       p_global=w.P, dl_rows=take, n_threads=NCPU, unscaled=True)
    check_seq(out.seq_logp.cpu().numpy()[seqs], o["seq_logp"], w.dtype)
    gi = torch.from_numpy(seqs).cuda()
    check_dlogits(to_f64(out.dlogits[gi][:, :3].reshape(-1, w.V)), o["dlogits"], 1.0, w.dtype)
    check_row_scale(out.row_scale[gi].cpu().numpy(), o["row_scale"], w.dtype)
    s = out.dlogits[:, :4].float().sum(dim=2)
    assert float(s.abs().max()) < 0.02
    seq, stats = out.seq_logp.clone(), out.stats[:10].clone()
    del out
    e = odpo.online_dpo_loss_fwd_bwd_unscaled(b.d_logits, ref, b.d_tokens, b.d_mask, w.beta,
                                              inplace=True)
    torch.cuda.synchronize()
    assert torch.allclose(e.seq_logp, seq, rtol=2e-5, atol=1e-3)
    assert abs(float(e.stats[1]) - float(stats[1])) <= 1e-5 * abs(float(stats[1])) + 1e-7
    del b, e
    torch.cuda.empty_cache()
