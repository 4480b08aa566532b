"""GPU-vs-oracle parity of the factored-gradient call (odpo_online_dpo_loss_fwd_bwd_unscaled,
SURVEY.md §8(b) performance tier): G = mask (softmax - onehot) and row_scale = coef_b mask,
against oracle.online_dpo_loss_fwd_bwd(..., unscaled=True) on the same seeded inputs."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_helpers import DL_RTOL, NCPU, Batch, alloc_rows, check_dlogits, check_seq, check_stats, to_f64

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def odpo():
    import paper_2410_18252_b200 as m
    m._L()
    return m


def run_unscaled(odpo, b: Batch, ref, beta, Pg=None, **kw):
    if not kw.get("inplace"):
        kw.setdefault("G", b.new_out())
    try:
        out = odpo.online_dpo_loss_fwd_bwd_unscaled(b.d_logits, ref, b.d_tokens, b.d_mask, beta,
                                                    pair_rows=b.d_pair_rows, p_global=Pg,
                                                    inv_temperature=b.invT, **kw)
    except odpo.OdpoError as e:
        # RESIDENT is compiled only in the experimental build (--odpo-lib ...experimental.so)
        if kw.get("schedule") == "resident" and "unsupported" in str(e):
            pytest.skip(f"resident schedule not in this build: {e}")
        raise
    torch.cuda.synchronize()
    return out


def check_row_scale(rs_gpu, rs_orc, dtype):
    rs_gpu = np.asarray(rs_gpu, dtype=np.float64)
    assert np.array_equal(rs_gpu == 0, rs_orc == 0), "row_scale zero pattern"
    assert np.all(np.sign(rs_gpu) == np.sign(rs_orc))
    err = np.abs(rs_gpu - rs_orc)
    assert np.all(err <= DL_RTOL[dtype] * np.abs(rs_orc)), f"row_scale max err {err.max():.3e}"


CASES = [
    # (P, T, V, dtype, mask, extra_seqs, invT) -- ragged tails, unreferenced sequences
    (3, 5, 4133, "bf16", "prefix", 2, 1.0),
    (3, 5, 4133, "f32", "prefix", 1, 1 / 0.7),
    (2, 9, 8, "bf16", "dense", 1, 1.0),
    (5, 17, 32000, "bf16", "prefix", 0, 1.0),
    (2, 7, 12345, "f32", "dense", 0, 1.0),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"P{c[0]}T{c[1]}V{c[2]}{c[3]}{c[4]}x{c[5]}")
@pytest.mark.parametrize("engine,row_gap,sched", [(-1, -1, "auto"), (0, 1, "auto"), (1, 0, "auto"),
                                                  (-1, -1, "resident")])
def test_unscaled_parity_small(odpo, case, engine, row_gap, sched):
    """sched "resident": each row's backward read back from tensor memory (k_resident, UN)."""
    P, T, V, dt, mk, extra, invT = case
    b = Batch(P, T, V, dt, seed=2, mask_kind=mk, lbar=max(1, T // 2), extra_seqs=extra, invT=invT)
    ref = (synth.rewards_for(2, b.B, 1).reshape(-1) - 30.0).astype(np.float32)
    beta, Pg = 0.1, P + 3
    d_ref = torch.from_numpy(ref).cuda()
    out = run_unscaled(odpo, b, d_ref, beta, Pg=Pg, engine=engine, row_gap=row_gap, schedule=sched)
    o = oracle.online_dpo_loss_fwd_bwd(b.h_logits, ref, b.tokens, b.mask, beta,
                                       pair_rows=b.pair_rows, p_global=Pg, inv_temperature=invT,
                                       want_dlogits=True, n_threads=NCPU, unscaled=True)
    live = np.arange(b.B) if b.pair_rows is None else b.pair_rows.reshape(-1)
    check_seq(out.seq_logp.cpu().numpy()[live], o["seq_logp"][live], dt)
    check_dlogits(to_f64(out.dlogits), o["dlogits"], 1.0, dt)
    check_row_scale(out.row_scale.cpu().numpy(), o["row_scale"], dt)
    check_stats(out.stats.cpu().numpy(), o, dt, beta, ref, b.pair_rows, Pg=Pg)
    assert int(out.status.item()) == 0
    # the loss outputs are the scaled call's, bit for bit (same rows, same reduction trees)
    sc = odpo.online_dpo_loss_fwd_bwd(b.d_logits, d_ref, b.d_tokens, b.d_mask, beta,
                                      pair_rows=b.d_pair_rows, p_global=Pg, inv_temperature=invT,
                                      dlogits=b.new_out(), engine=max(engine, 0))
    torch.cuda.synchronize()
    assert torch.equal(sc.seq_logp[live], out.seq_logp[live])
    assert torch.equal(sc.z, out.z)
    assert torch.equal(sc.stats[:10], out.stats[:10])
    # row_scale * G reproduces dlogits (both roundings of one exact value: 2 ulps)
    prod = out.row_scale.double()[..., None] * out.dlogits.double()
    ref_dl = sc.dlogits.double()
    tol = (2 * DL_RTOL[dt]) * ref_dl.abs() + 1e-30 + 2.0 ** -20 * out.row_scale.double().abs()[..., None]
    assert bool(((prod - ref_dl).abs() <= tol).all())


def test_unscaled_inplace_and_deterministic(odpo):
    P, T, V = 6, 13, 9001
    b = Batch(P, T, V, "bf16", seed=8, mask_kind="prefix", lbar=7, host=False)
    ref = torch.full((b.B,), -10.0, device="cuda")
    a1 = run_unscaled(odpo, b, ref, 0.1)
    a2 = run_unscaled(odpo, b, ref, 0.1)
    assert torch.equal(a1.dlogits, a2.dlogits) and torch.equal(a1.row_scale, a2.row_scale)
    x = alloc_rows(b.B, b.T, b.V, "bf16")
    x.copy_(b.d_logits)
    bi = Batch.__new__(Batch)
    bi.__dict__.update(b.__dict__)
    bi.d_logits = x
    a3 = run_unscaled(odpo, bi, ref, 0.1, inplace=True)
    assert a3.dlogits.data_ptr() == x.data_ptr()
    assert torch.equal(a3.dlogits, a1.dlogits) and torch.equal(a3.row_scale, a1.row_scale)
    assert torch.equal(a3.stats, a1.stats)


def test_best_worst_of_k4_workload(odpo):
    """NEXT-1 shape (App A.3 617/632-633): K = 4 completions per prompt, binary
    verifier rewards, pair_select picks 2 of 4; the 2 unselected completions of every prompt
    are unreferenced sequences: G = 0 and row_scale = 0 on their rows."""
    P, K, T, V = 16, 4, 9, 3001
    rewards = synth.rewards_for(6, P, K, kind="verifier")
    eos = synth.has_eos_for(6, P, K)
    sel = odpo.pair_select(torch.from_numpy(rewards).cuda(), torch.from_numpy(eos).cuda(), -1.0)
    o_sel = oracle.pair_select(rewards, eos, -1.0)
    assert np.array_equal(sel.pair_rows.cpu().numpy(), o_sel["pair_rows"])
    b = Batch(P, T, V, "bf16", seed=6, mask_kind="prefix", lbar=5, extra_seqs=(K - 2) * P)
    b.pair_rows = o_sel["pair_rows"].astype(np.int32)
    b.d_pair_rows = sel.pair_rows
    ref = np.full(b.B, -0.5 * T, np.float32)
    out = run_unscaled(odpo, b, torch.from_numpy(ref).cuda(), 0.1)
    try:
        res = odpo.online_dpo_loss_fwd_bwd_unscaled(
            b.d_logits, torch.from_numpy(ref).cuda(), b.d_tokens, b.d_mask, 0.1,
            pair_rows=b.d_pair_rows, G=b.new_out(), schedule="resident")
        torch.cuda.synchronize()
        assert torch.equal(res.dlogits, out.dlogits) and torch.equal(res.row_scale, out.row_scale)
    except odpo.OdpoError as e:
        assert "unsupported" in str(e)   # not in this build
    o = oracle.online_dpo_loss_fwd_bwd(b.h_logits, ref, b.tokens, b.mask, 0.1,
                                       pair_rows=b.pair_rows, want_dlogits=True, n_threads=NCPU,
                                       unscaled=True)
    check_dlogits(to_f64(out.dlogits), o["dlogits"], 1.0, "bf16")
    check_row_scale(out.row_scale.cpu().numpy(), o["row_scale"], "bf16")
    unref = np.setdiff1d(np.arange(b.B), b.pair_rows.reshape(-1))
    assert len(unref) == (K - 2) * P
    assert torch.count_nonzero(out.dlogits[torch.from_numpy(unref).cuda()]).item() == 0


@pytest.mark.parametrize("name,mask_kind", [("pythia", "dense"), ("llama", "prefix")])
def test_unscaled_full_size_sampled(odpo, name, mask_kind):
    """BASELINE.json configs at full size in the bench's launch configuration: sampled rows
    against the oracle; loss outputs equal to the scaled call's."""
    from synth.configs import CONFIGS
    w = CONFIGS[name]
    b = Batch(w.P, w.T, w.V, w.dtype, seed=0, mask_kind=mask_kind, lbar=w.lbar, host=False)
    ref = torch.full((b.B,), -float(w.T) * 0.08, dtype=torch.float32, device="cuda")
    out = run_unscaled(odpo, b, ref, w.beta)
    seq = out.seq_logp.clone()
    z = out.z.clone()
    stats = out.stats[:10].clone()
    pairs = synth.permutation(1, w.P)[:2]
    seqs = np.stack([2 * pairs, 2 * pairs + 1], 1).reshape(-1)
    h_x = b.host_rows(seqs)
    h_ref = np.full(len(seqs), -float(w.T) * 0.08, np.float32)
    rows = (np.arange(len(seqs))[:, None] * w.T + np.arange(w.T)[None, :])
    take = rows[:, :3].reshape(-1)
    o = oracle.online_dpo_loss_fwd_bwd(h_x, h_ref, b.tokens[seqs], b.mask[seqs], w.beta,
                                       p_global=w.P, dl_rows=take, n_threads=NCPU, unscaled=True)
    check_seq(seq.cpu().numpy()[seqs], o["seq_logp"], w.dtype)
    gi = torch.from_numpy(seqs).cuda()
    g = to_f64(out.dlogits[gi][:, :3].reshape(-1, w.V))
    check_dlogits(g, o["dlogits"], 1.0, w.dtype)
    check_row_scale(out.row_scale[gi].cpu().numpy(), o["row_scale"], w.dtype)
    assert int(out.status.item()) == 0
    # every live row of G sums to ~0 (softmax sums to 1): a property at any size
    s = out.dlogits[:, :4].float().sum(dim=2)
    assert float(s.abs().max()) < 0.02
    if w.V * 2 <= (128 << 10):
        # the RESIDENT factored gradient (rows read back from TMEM) gives the same bits
        try:
            res = odpo.online_dpo_loss_fwd_bwd_unscaled(b.d_logits, ref, b.d_tokens, b.d_mask,
                                                        w.beta, G=b.new_out(), schedule="resident")
            torch.cuda.synchronize()
            assert torch.equal(res.dlogits, out.dlogits) and torch.equal(res.row_scale, out.row_scale)
            assert torch.equal(res.seq_logp, seq) and torch.equal(res.stats[:10], stats)
            del res
        except odpo.OdpoError as e:
            assert "unsupported" in str(e)   # RESIDENT is in the experimental build only
    del out
    # same engine geometry as the unscaled call's automatic choice (the geometry fixes the
    # per-row reduction tree): geometry 1 for rows longer than 128 KB
    geo = 1 if w.V * 2 > (128 << 10) else 0
    sc = odpo.online_dpo_loss_fwd_bwd(b.d_logits, ref, b.d_tokens, b.d_mask, w.beta, inplace=True,
                                      engine=geo)
    torch.cuda.synchronize()
    assert torch.equal(sc.seq_logp, seq) and torch.equal(sc.z, z)
    assert torch.equal(sc.stats[:10], stats)
    del b, sc
    torch.cuda.empty_cache()
