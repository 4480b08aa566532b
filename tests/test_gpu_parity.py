"""GPU-vs-oracle parity of the CUDA path through the C ABI.

Every input is drawn from ``synth`` (seeded, synthetic, shaped like the paper's
workloads); the oracle never sees a value produced by the CUDA path except the
explicitly-constructed "controlled ref" inputs, which are inputs to both sides."""
import math
import struct

import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_helpers import (NCPU, Batch, alloc_rows, check_dlogits, check_seq, check_stats,
                         coef_from_oracle, to_f64)

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

SCHEDS = ["fused", "two_pass", "wave", "resident", "psync"]
OPTIONAL = ("resident", "psync")   # schedules that apply to some shapes only (odpo.h)


@pytest.fixture(scope="module")
def odpo():
    import paper_2410_18252_b200 as m
    m._L()
    return m


def run_loss(odpo, b: Batch, ref, beta, sched="fused", Pg=None, **kw):
    if not kw.get("inplace"):
        kw.setdefault("dlogits", b.new_out())
    try:
        out = odpo.online_dpo_loss_fwd_bwd(b.d_logits, ref, b.d_tokens, b.d_mask, beta,
                                           pair_rows=b.d_pair_rows, p_global=Pg,
                                           inv_temperature=b.invT, schedule=sched, **kw)
    except odpo.OdpoError as e:
        # the RESIDENT schedule applies only where two rows fit in shared memory and the
        # on-chip stash holds two pairs (odpo.h); elsewhere the library refuses it
        if sched in OPTIONAL and "unsupported" in str(e):
            pytest.skip(f"{sched} schedule does not apply: {e}")
        raise
    torch.cuda.synchronize()
    return out


def oracle_loss(b: Batch, ref, beta, Pg=None, want_dlogits=True):
    return oracle.online_dpo_loss_fwd_bwd(b.h_logits, ref, b.tokens, b.mask, beta,
                                          pair_rows=b.pair_rows, p_global=Pg,
                                          inv_temperature=b.invT, want_dlogits=want_dlogits,
                                          n_threads=NCPU)


# ------------------------------------------------------------------------ synth twin
def test_device_generator_matches_host_twin():
    b = Batch(2, 3, 1000, "bf16", seed=5, p0=7, host=True)
    dev_bits = b.d_logits.view(torch.int16).cpu().numpy().view(np.uint16)
    assert np.array_equal(dev_bits, b.h_logits)
    b = Batch(1, 2, 515, "f32", seed=9, host=True, peak=None)
    assert np.array_equal(b.d_logits.cpu().numpy(), b.h_logits)


# ------------------------------------------------------------------------ G-1 pair_select
@pytest.mark.parametrize("K", [2, 3, 4])
def test_pair_select_bit_exact(odpo, K):
    vals = [-1.0, 0.0, 0.5, 1.0]
    import itertools
    ex = np.array(list(itertools.product(vals, repeat=K)), dtype=np.float32)
    rnd = synth.rewards_for(3, 2048, K)
    for rewards, eos, pen in [(ex, None, -1.0), (rnd, synth.has_eos_for(3, 2048, K), -10.0),
                              (synth.rewards_for(4, 2048, K, kind="verifier"), None, -1.0)]:
        d_eos = None if eos is None else torch.from_numpy(eos).cuda()
        g = odpo.pair_select(torch.from_numpy(rewards).cuda(), d_eos, pen)
        o = oracle.pair_select(rewards, eos, pen)
        assert np.array_equal(g.chosen.cpu().numpy(), o["chosen"])
        assert np.array_equal(g.rejected.cpu().numpy(), o["rejected"])
        assert np.array_equal(g.pair_rows.cpu().numpy(), o["pair_rows"])
        assert np.array_equal(g.reward_margin.cpu().numpy().view(np.uint32),
                              o["margin"].view(np.uint32))
        s = g.sel_stats.cpu().numpy()
        assert s[1] == o["sel_stats"][1] and s[2] == o["sel_stats"][2]
        assert abs(s[0] - o["sel_stats"][0]) <= 1e-12 * max(1.0, abs(o["sel_stats"][0]))
        assert int(g.status.item()) == o["status"]


def test_pair_select_spec_margin_bits(odpo):
    g = odpo.pair_select(torch.tensor([[0.9, 0.1], [0.1, 0.9]], dtype=torch.float32).cuda())
    assert g.reward_margin.cpu().numpy().view(np.uint32).tolist() == [0x3F4CCCCC] * 2
    assert g.chosen.tolist() == [0, 1]


# ------------------------------------------------------------------------ G-2 identity rows
def identity_batch(P, T, V, dtype, seed, permute):
    """Anchor construction (SURVEY §8(c) 'GPU indexing'): every per-token log-prob is
    exactly -(c + 100), so routing/gather/pairing errors change bits."""
    B = 2 * P + (2 if permute else 0)
    tok = synth.tokens_rows(seed, np.arange(B * T), V).reshape(B, T)
    c = 1.0 + (synth.uniform_u32(seed, 11, np.arange(B * T)) % 64).astype(np.float64) / 8.0
    x = np.zeros((B, T, V))
    bi, ti = np.meshgrid(np.arange(B), np.arange(T), indexing="ij")
    x[bi, ti, (tok + 1) % V] = 100.0
    x[bi, ti, tok] = -c.reshape(B, T)
    mask = synth.mask_for(seed, np.arange(B), T, "prefix", max(1, T // 2))
    pr = synth.permutation(seed, B)[: 2 * P].reshape(P, 2).astype(np.int32) if permute else None
    # ref = S_b + offset on the 1/8 grid, so z is moderate (sigma(-z) does not underflow)
    # and still exact in fp32
    S = np.where(mask == 1, -c.reshape(B, T) - 100.0, 0.0).sum(1)
    off = (synth.uniform_u32(seed, 12, np.arange(B)) % 64).astype(np.float64) / 8.0 - 4.0
    return x, tok.astype(np.int32), mask, pr, (S + off).astype(np.float32)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("permute", [False, True])
@pytest.mark.parametrize("sched", SCHEDS)
@pytest.mark.parametrize("shape", [(4, 53, 50304), (3, 5, 1003)])
def test_identity_rows_bit_exact(odpo, dtype, permute, sched, shape):
    P, T, V = shape
    x, tok, mask, pr, ref = identity_batch(P, T, V, dtype, 1, permute)
    B = x.shape[0]
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    d_x = alloc_rows(B, T, V, dtype)
    d_x.copy_(torch.from_numpy(x.astype(np.float32)).cuda().to(tdt))
    h_x = x.astype(np.float32) if dtype == "f32" else oracle.to_bf16_bits(x)
    beta = 0.125
    try:
        out = odpo.online_dpo_loss_fwd_bwd(
            d_x, torch.from_numpy(ref).cuda(), torch.from_numpy(tok).cuda(),
            torch.from_numpy(mask).cuda(), beta,
            pair_rows=None if pr is None else torch.from_numpy(pr).cuda(), schedule=sched,
            dlogits=alloc_rows(B, T, V, dtype))
    except odpo.OdpoError as e:
        if sched in OPTIONAL and "unsupported" in str(e):
            pytest.skip(f"{sched} schedule does not apply: {e}")
        raise
    torch.cuda.synchronize()
    o = oracle.online_dpo_loss_fwd_bwd(h_x, ref, tok, mask, beta, pair_rows=pr, n_threads=NCPU)
    # per-sequence log-probs and z are exact (1/8-grid arithmetic)
    S_exp = -(np.where(mask == 1, -x[np.arange(B)[:, None], np.arange(tok.shape[1])[None, :], tok] + 100.0, 0.0)).sum(1)
    seq_gpu = out.seq_logp.cpu().numpy()
    ref_idx = np.arange(B) if pr is None else pr.reshape(-1)
    assert np.array_equal(seq_gpu[ref_idx].astype(np.float64), o["seq_logp"][ref_idx])
    assert np.array_equal(seq_gpu[ref_idx].astype(np.float64), S_exp[ref_idx])
    assert np.array_equal(out.z.cpu().numpy().astype(np.float64), o["z"])
    # statistics: S, ref, beta = 1/8 and z are exact, so every margin statistic is too
    st = out.stats.cpu().numpy()
    for i in (0, 2, 3, 4, 5, 6, 7, 8, 9):
        assert st[i] == o["stats"][i], (i, st[i], o["stats"][i])
    assert abs(st[1] - o["stats"][1]) <= 1e-6 * abs(o["stats"][1])
    # dlogits pattern: exactly two nonzeros per live row, +coef at the anchor, -coef at tok
    g = out.dlogits.float().cpu().numpy()
    seq_role = {}
    for p in range(P):
        cc, rr = (2 * p, 2 * p + 1) if pr is None else pr[p]
        seq_role[int(cc)] = p
        seq_role[int(rr)] = p
    for b in range(B):
        for t in range(tok.shape[1]):
            row = g[b, t]
            if b not in seq_role or not mask[b, t]:
                assert not np.any(row), (b, t)
                continue
            # entries above 2^-20 |coef|: underflowed softmax terms are exactly 0 on the MUFU
            # path and <= 2^-125 |coef| on the FMA-polynomial exp2 path
            big = 2.0 ** -20 * np.max(np.abs(row))
            nz = np.flatnonzero(np.abs(row) > big)
            a = (tok[b, t] + 1) % V
            assert sorted(nz.tolist()) == sorted([a, tok[b, t]]), (b, t, nz[:5])
            # +coef at the anchor (softmax 1 up to the fp32 rounding of m*invT*log2e) and
            # -coef at tok (expm1(-(c+100)) = -1 exactly)
            assert abs(row[a] + row[tok[b, t]]) <= 2.0 ** -7 * abs(row[tok[b, t]])  # 1 bf16 ulp (R17)


# ------------------------------------------------------------------------ G-3/4/5 parity
CASES = [
    # (P, T, V, dtype, mask, extra_seqs, invT)  -- several tiles + ragged vocabulary tails
    (3, 5, 4133, "bf16", "prefix", 2, 1.0),
    (3, 5, 4133, "f32", "prefix", 0, 1 / 0.7),
    (2, 9, 8, "bf16", "dense", 1, 1.0),
    (5, 17, 32000, "bf16", "prefix", 0, 1.0),
    (2, 7, 12345, "f32", "dense", 0, 1.0),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"P{c[0]}T{c[1]}V{c[2]}{c[3]}{c[4]}x{c[5]}")
@pytest.mark.parametrize("sched", SCHEDS)
def test_loss_parity_small(odpo, case, sched):
    P, T, V, dt, mk, extra, invT = case
    b = Batch(P, T, V, dt, seed=2, mask_kind=mk, lbar=max(1, T // 2), extra_seqs=extra, invT=invT)
    ref = (synth.rewards_for(2, b.B, 1).reshape(-1) - 30.0).astype(np.float32)
    beta = 0.1
    out = run_loss(odpo, b, torch.from_numpy(ref).cuda(), beta, sched, Pg=P + 3)
    o = oracle_loss(b, ref, beta, Pg=P + 3)
    live = np.arange(b.B) if b.pair_rows is None else b.pair_rows.reshape(-1)
    check_seq(out.seq_logp.cpu().numpy()[live], o["seq_logp"][live], dt)
    check_stats(out.stats.cpu().numpy(), o, dt, beta, ref, b.pair_rows, Pg=P + 3)
    coef = coef_from_oracle(o, P, P + 3, beta, invT, b.pair_rows, b.B)
    check_dlogits(to_f64(out.dlogits), o["dlogits"], coef[:, None, None], dt)


@pytest.mark.parametrize("case", CASES[:2] + CASES[3:4], ids=lambda c: f"P{c[0]}V{c[2]}{c[3]}")
@pytest.mark.parametrize("sched", SCHEDS)
def test_loss_parity_engine_geometry1(odpo, case, sched):
    """The same parity with the large-row engine geometry (8 warps x 6 stages x 2 CTAs/SM)."""
    P, T, V, dt, mk, extra, invT = case
    b = Batch(P, T, V, dt, seed=5, mask_kind=mk, lbar=max(1, T // 2), extra_seqs=extra, invT=invT)
    ref = (synth.rewards_for(5, b.B, 1).reshape(-1) - 30.0).astype(np.float32)
    out = run_loss(odpo, b, torch.from_numpy(ref).cuda(), 0.1, sched, engine=1)
    o = oracle_loss(b, ref, 0.1)
    live = np.arange(b.B) if b.pair_rows is None else b.pair_rows.reshape(-1)
    check_seq(out.seq_logp.cpu().numpy()[live], o["seq_logp"][live], dt)
    coef = coef_from_oracle(o, P, P, 0.1, invT, b.pair_rows, b.B)
    check_dlogits(to_f64(out.dlogits), o["dlogits"], coef[:, None, None], dt)
    # the geometry fixes the per-row reduction tree (warps per CTA): deterministic per geometry
    again = run_loss(odpo, b, torch.from_numpy(ref).cuda(), 0.1, sched, engine=1)
    li = torch.from_numpy(live).cuda()
    assert torch.equal(again.seq_logp[li], out.seq_logp[li])
    assert torch.equal(again.dlogits, out.dlogits)


@pytest.mark.parametrize("sched", SCHEDS)
def test_tiny_config_full_parity(odpo, sched):
    """BASELINE.json configs[0]: 4 prompts x 2, T=53, V=50304, fp32, beta=0.05 (full dlogits)."""
    from synth.configs import CONFIGS
    w = CONFIGS["tiny"]
    b = Batch(w.P, w.T, w.V, w.dtype, seed=0)
    rewards = synth.rewards_for(0, w.P, 2)
    eos = synth.has_eos_for(0, w.P, 2)
    sel = odpo.pair_select(torch.from_numpy(rewards).cuda(), torch.from_numpy(eos).cuda(), w.eos_penalty)
    o_sel = oracle.pair_select(rewards, eos, w.eos_penalty)
    assert np.array_equal(sel.pair_rows.cpu().numpy(), o_sel["pair_rows"])
    b.pair_rows = o_sel["pair_rows"]
    b.d_pair_rows = sel.pair_rows
    # realistic ref: an independent "reference model" (seed+1 logits), through the oracle
    h_ref = synth.logits_rows(0, b.rows_global, w.V, tokens=b.tokens.reshape(-1), peak=14.0,
                              ref=True).reshape(b.B, w.T, w.V).astype(np.float32)
    ref = oracle.seq_logprobs(h_ref, b.tokens, b.mask, n_threads=NCPU)["seq_logp"].astype(np.float32)
    out = run_loss(odpo, b, torch.from_numpy(ref).cuda(), w.beta, sched)
    o = oracle_loss(b, ref, w.beta)
    check_seq(out.seq_logp.cpu().numpy(), o["seq_logp"], "f32")
    check_stats(out.stats.cpu().numpy(), o, "f32", w.beta, ref, b.pair_rows)
    coef = coef_from_oracle(o, w.P, w.P, w.beta, 1.0, b.pair_rows, b.B)
    check_dlogits(to_f64(out.dlogits), o["dlogits"], coef[:, None, None], "f32")
    # ref pass through the GPU seq_logprobs on the device-generated ref logits
    d_ref_logits = torch.empty_like(b.d_logits)
    synth.fill_logits_device(d_ref_logits, 0, row0=0, tokens=b.d_tokens, peak=14.0, ref=True)
    g_ref = odpo.seq_logprobs(d_ref_logits, b.d_tokens, b.d_mask)
    torch.cuda.synchronize()
    check_seq(g_ref.cpu().numpy(), ref.astype(np.float64), "f32", "ref seq_logp")


def test_controlled_ref_accuracy_exact(odpo):
    """Controlled-ref mode: ref = fl32(S_gpu - delta), |z| >= beta/16, so the
    accuracy count must match the oracle exactly."""
    P, T, V = 64, 11, 5000
    b = Batch(P, T, V, "bf16", seed=3, mask_kind="prefix", lbar=6)
    S = odpo.seq_logprobs(b.d_logits, b.d_tokens, b.d_mask).cpu().numpy()
    h = synth.uniform_u32(3, synth.S_DELTA, np.arange(P))
    delta = np.zeros(2 * P, np.float32)
    delta[0::2] = np.where(h & 1, 1.0, -1.0) * (1 + (h >> 1) % 128) / 16.0
    ref = (S - delta).astype(np.float32)
    beta = 0.03
    out = run_loss(odpo, b, torch.from_numpy(ref).cuda(), beta)
    o = oracle_loss(b, ref, beta, want_dlogits=False)
    st = out.stats.cpu().numpy()
    assert st[2] == o["stats"][2]
    assert 0 < st[2] < P
    check_stats(st, o, "bf16", beta, ref, None, exact_ncorrect=True)
    zg = out.z.cpu().numpy().astype(np.float64)
    assert np.all(np.sign(zg) == np.sign(o["z"]))


# ------------------------------------------------------------------------ full-size sampled parity
FULL = [("pythia", "dense", 4), ("rho", "dense", 2), ("llama", "prefix", 2)]


@pytest.mark.parametrize("name,mask_kind,nsample", FULL)
def test_full_size_sampled_parity(odpo, name, mask_kind, nsample):
    """BASELINE.json configs at full size, in the launch configuration bench.py times
    (fused schedule, default lag): sampled pairs against the oracle, global stats via
    properties that hold at any size."""
    from synth.configs import CONFIGS
    w = CONFIGS[name]
    b = Batch(w.P, w.T, w.V, w.dtype, seed=0, mask_kind=mask_kind, lbar=w.lbar, host=False)
    ref = torch.full((b.B,), -float(w.T) * 0.08, dtype=torch.float32, device="cuda")
    out = run_loss(odpo, b, ref, w.beta, "fused", inplace=False)
    two = run_loss(odpo, b, ref, w.beta, "two_pass")
    # both schedules share the per-row arithmetic and reduction trees: bit-identical
    assert torch.equal(out.seq_logp, two.seq_logp)
    assert torch.equal(out.z, two.z)
    assert torch.equal(out.stats[:10], two.stats[:10])
    del two
    # the wave schedule (pairs pinned to CTA groups) gives the same bits, dlogits included
    auto = run_loss(odpo, b, ref, w.beta, "wave" if 2 * w.T <= 148 * 4 else "auto")
    assert torch.equal(auto.seq_logp, out.seq_logp) and torch.equal(auto.stats[:10], out.stats[:10])
    assert torch.equal(auto.dlogits, out.dlogits)
    del auto
    # the RESIDENT schedule (rows kept on chip; AUTO for the Pythia shape): same parity bar
    outs = {"fused": out}
    try:
        outs["resident"] = odpo.online_dpo_loss_fwd_bwd(
            b.d_logits, ref, b.d_tokens, b.d_mask, w.beta, pair_rows=b.d_pair_rows,
            schedule="resident", dlogits=b.new_out())
        torch.cuda.synchronize()
        res = outs["resident"]
        assert int(res.status.item()) == int(out.status.item())
        # the same per-row reduction tree as FUSED (4 forward warps x 8 vectors per chunk):
        # row statistics, sequence sums, loss and dlogits are bit-identical
        assert torch.equal(res.seq_logp, out.seq_logp) and torch.equal(res.z, out.z)
        assert torch.equal(res.stats[:10], out.stats[:10])
        assert torch.equal(res.dlogits, out.dlogits)
    except odpo.OdpoError as e:
        # RESIDENT is compiled only in the experimental build; there it applies to Pythia
        assert "unsupported" in str(e)
    pairs = synth.permutation(1, w.P)[:nsample]
    seqs = np.stack([2 * pairs, 2 * pairs + 1], 1).reshape(-1)
    h_x = b.host_rows(seqs)
    sub_tok = b.tokens[seqs]
    sub_mask = b.mask[seqs]
    h_ref = np.full(len(seqs), -float(w.T) * 0.08, np.float32)
    rows = (np.arange(len(seqs))[:, None] * w.T + np.arange(w.T)[None, :]).reshape(-1)
    # dlogits for a bounded subset of rows (the first rows of each sampled sequence)
    take = rows.reshape(len(seqs), w.T)[:, :3].reshape(-1)
    o = oracle.online_dpo_loss_fwd_bwd(h_x, h_ref, sub_tok, sub_mask, w.beta, p_global=w.P,
                                       dl_rows=take, n_threads=NCPU)
    for out in outs.values():
        check_seq(out.seq_logp.cpu().numpy()[seqs], o["seq_logp"], w.dtype)
        zg = out.z.cpu().numpy()[pairs].astype(np.float64)
        assert np.all(np.abs(zg - o["z"]) <= 2e-3 * np.maximum(np.abs(o["z"]), 1.0))
        gi = torch.from_numpy(seqs).cuda()
        g = to_f64(out.dlogits[gi][:, :3].reshape(-1, w.V))
        coef = np.repeat(coef_from_oracle(o, nsample, w.P, w.beta, 1.0, None, len(seqs)), 3)
        check_dlogits(g, o["dlogits"], coef[:, None], w.dtype)
    del outs
    # global stats: properties of the GPU's own per-pair outputs (any size)
    z_all = out.z.cpu().double().numpy()
    st = out.stats.cpu().numpy()
    loss = np.sum(np.maximum(-z_all, 0) + np.log1p(np.exp(-np.abs(z_all)))) / w.P
    assert abs(st[1] - loss) <= 1e-9 * max(abs(loss), 1e-6)
    assert st[0] == w.P and st[2] == np.count_nonzero(z_all > 0)
    assert st[8] + st[9] == b.mask.sum()
    # margin statistics: z_sum is the sum of the published z; the implicit rewards and the
    # sequence sums are those of the published seq_logp (any summation order: 1e-9 relative)
    S_all = out.seq_logp.cpu().double().numpy()
    rf = ref.cpu().double().numpy()
    sz = np.abs(z_all).sum()
    assert abs(st[3] - z_all.sum()) <= 1e-9 * max(sz, 1e-9)
    Sc, Sr = S_all[0::2], S_all[1::2]
    bt = float(np.float32(w.beta))
    assert abs(st[6] - Sc.sum()) <= 1e-9 * np.abs(Sc).sum()
    assert abs(st[7] - Sr.sum()) <= 1e-9 * np.abs(Sr).sum()
    dc = (Sc.astype(np.float32) - rf[0::2].astype(np.float32)).astype(np.float64)
    dr = (Sr.astype(np.float32) - rf[1::2].astype(np.float32)).astype(np.float64)
    assert abs(st[4] - bt * dc.sum()) <= 1e-9 * bt * np.abs(dc).sum() + 1e-12
    assert abs(st[5] - bt * dr.sum()) <= 1e-9 * bt * np.abs(dr).sum() + 1e-12
    assert abs(st[3] - (st[4] - st[5])) <= 2.0 ** -23 * sz + 1e-9 * bt * (np.abs(dc).sum() + np.abs(dr).sum())
    assert int(out.status.item()) == 0
    del b, out
    torch.cuda.empty_cache()


# ------------------------------------------------------------------------ G-6 self-consistency
@pytest.mark.parametrize("sched", SCHEDS)
def test_self_consistency_ln2(odpo, sched):
    P, T, V = 16, 9, 7777
    b = Batch(P, T, V, "bf16", seed=4, mask_kind="prefix", lbar=5, host=False)
    S = odpo.seq_logprobs(b.d_logits, b.d_tokens, b.d_mask)
    out = run_loss(odpo, b, S.clone(), 0.1, sched)
    assert torch.equal(out.seq_logp, S)
    assert torch.count_nonzero(out.z).item() == 0
    st = out.stats.cpu().numpy()
    assert abs(st[1] - math.log(2.0)) < 1e-12 and st[2] == 0.0


# ------------------------------------------------------------------------ G-7 poison
def test_poisoned_rows(odpo):
    P, T, V = 3, 6, 3001
    b = Batch(P, T, V, "bf16", seed=6, mask_kind="prefix", lbar=3, host=False)
    ref = torch.zeros(b.B, device="cuda")
    clean = run_loss(odpo, b, ref, 0.1)
    dl_clean = clean.dlogits.clone()
    live = b.mask == 1
    dead = np.argwhere(~live)
    assert len(dead) > 0
    x = b.d_logits
    for k, (s, t) in enumerate(dead[:4]):
        x[s, t, (17 * k) % V] = float("nan") if k % 2 else float("inf")
    dirty = run_loss(odpo, b, ref, 0.1)
    assert int(dirty.status.item()) == 0
    assert torch.equal(dirty.seq_logp, clean.seq_logp)
    assert torch.equal(dirty.dlogits, dl_clean)
    s, t = np.argwhere(live)[0]
    x[s, t, 5] = float("nan")
    assert int(run_loss(odpo, b, ref, 0.1).status.item()) & odpo.FLAGS["NONFINITE_LOGIT"]
    x[s, t, 5] = float("inf")
    assert int(run_loss(odpo, b, ref, 0.1).status.item()) & odpo.FLAGS["NONFINITE_LOGIT"]
    x[s, t, 5] = float("-inf")   # legal (R14) unless it is the sampled token
    if b.tokens[s, t] != 5:
        assert int(run_loss(odpo, b, ref, 0.1).status.item()) == 0
    tk = b.d_tokens.clone()
    b.d_tokens[s, t] = V
    assert int(run_loss(odpo, b, ref, 0.1).status.item()) & odpo.FLAGS["TOKEN_RANGE"]
    b.d_tokens.copy_(tk)
    b.d_tokens[s, t] = -1
    assert int(run_loss(odpo, b, ref, 0.1).status.item()) & odpo.FLAGS["TOKEN_RANGE"]
    b.d_tokens.copy_(tk)
    m = b.d_mask.clone()
    b.d_mask[1] = 0
    o = run_loss(odpo, b, ref, 0.1)
    assert int(o.status.item()) & odpo.FLAGS["EMPTY_SEQ"] and o.seq_logp[1].item() == 0.0
    b.d_mask.copy_(m)
    dup = torch.tensor([[0, 1], [1, 2], [3, 4]], dtype=torch.int32, device="cuda")
    o = odpo.online_dpo_loss_fwd_bwd(b.d_logits, ref, b.d_tokens, b.d_mask, 0.1, pair_rows=dup,
                                     dlogits=b.new_out())
    assert int(o.status.item()) & odpo.FLAGS["DUP_ROW"]
    bad = torch.tensor([[0, 1], [2, 99], [3, 4]], dtype=torch.int32, device="cuda")
    o = odpo.online_dpo_loss_fwd_bwd(b.d_logits, ref, b.d_tokens, b.d_mask, 0.1, pair_rows=bad,
                                     dlogits=b.new_out())
    torch.cuda.synchronize()
    assert int(o.status.item()) & odpo.FLAGS["PAIR_RANGE"]


# ------------------------------------------------------------------------ G-8/9/10
@pytest.mark.parametrize("sched", SCHEDS)
def test_inplace_strided_deterministic(odpo, sched):
    P, T, V, Tp = 4, 7, 5000, 3
    b = Batch(P, T, V, "bf16", seed=8, mask_kind="prefix", lbar=4, host=False)
    ref = torch.full((b.B,), -2.0, device="cuda")
    base = run_loss(odpo, b, ref, 0.1, sched)
    again = run_loss(odpo, b, ref, 0.1, sched)
    assert torch.equal(base.dlogits, again.dlogits) and torch.equal(base.stats, again.stats)
    # strided view: logits live inside a longer [B, Tp + T, V] buffer
    big = torch.zeros((b.B, Tp + T, V), dtype=torch.bfloat16, device="cuda")
    big[:, Tp - 1:Tp - 1 + T].copy_(b.d_logits)
    view = big[:, Tp - 1:Tp - 1 + T]
    o = odpo.online_dpo_loss_fwd_bwd(view, ref, b.d_tokens, b.d_mask, 0.1, schedule=sched,
                                     dlogits=b.new_out())
    torch.cuda.synchronize()
    assert torch.equal(o.dlogits, base.dlogits) and torch.equal(o.stats, base.stats)
    # in place over the strided view
    o = odpo.online_dpo_loss_fwd_bwd(view, ref, b.d_tokens, b.d_mask, 0.1, schedule=sched, inplace=True)
    torch.cuda.synchronize()
    assert torch.equal(view, base.dlogits) and torch.equal(o.seq_logp, base.seq_logp)


# ------------------------------------------------------------------------ G-11 world size
@pytest.mark.parametrize("W", [2, 4, 8])
def test_world_size_invariance(odpo, W):
    """Contiguous pair shards with the static P_global reproduce the W=1 run: integer stats
    equal, float stats within fp64 rounding, dlogits rows bit-identical."""
    P, T, V = 16, 9, 6000
    full = Batch(P, T, V, "bf16", seed=10, mask_kind="prefix", lbar=5, host=False)
    ref = torch.linspace(-9, -1, full.B, device="cuda")
    one = run_loss(odpo, full, ref, 0.05)
    acc = torch.zeros(10, dtype=torch.float64)
    for r in range(W):
        p0, p1 = r * P // W, (r + 1) * P // W
        sh = Batch(p1 - p0, T, V, "bf16", seed=10, mask_kind="prefix", lbar=5, p0=p0, host=False)
        o = run_loss(odpo, sh, ref[2 * p0:2 * p1].contiguous(), 0.05, Pg=P)
        acc += o.stats[:10].cpu()
        assert torch.equal(o.dlogits, one.dlogits[2 * p0:2 * p1])
        assert torch.equal(o.z, one.z[p0:p1])
    s1 = one.stats[:10].cpu()
    for i in (0, 2, 8, 9):
        assert acc[i] == s1[i]
    assert torch.allclose(acc, s1, rtol=1e-12, atol=1e-12)


# ------------------------------------------------------------------------ seq_logprobs per token
def test_seq_logprobs_per_token(odpo):
    P, T, V = 3, 8, 3333
    b = Batch(P, T, V, "f32", seed=12, mask_kind="prefix", lbar=4, invT=1 / 0.7)
    seq, tok, lse, status = odpo.seq_logprobs(b.d_logits, b.d_tokens, b.d_mask, b.invT, per_token=True)
    torch.cuda.synchronize()
    o = oracle.seq_logprobs(b.h_logits, b.tokens, b.mask, b.invT)
    check_seq(seq.cpu().numpy(), o["seq_logp"], "f32")
    tg = tok.cpu().numpy().astype(np.float64)
    assert np.all(np.abs(tg - o["tok_logp"]) <= 1e-5 * np.maximum(np.abs(o["tok_logp"]), 1e-2))
    lg = lse.cpu().numpy().astype(np.float64)
    assert np.all(np.abs(lg - o["row_lse"]) <= 1e-6 * np.maximum(np.abs(o["row_lse"]), 1.0))
    assert np.all(tg[b.mask == 0] == 0)


# ------------------------------------------------------------------------ NEXT-1 gather
def test_gather_pairs_bit_exact(odpo):
    """K = 4: the selected completions compacted into pair order equal numpy fancy indexing
    of pair_select's rows; an out-of-range row is flagged and zeroed."""
    P, K, T = 63, 4, 37
    rewards = synth.rewards_for(3, P, K, kind="verifier")
    sel = odpo.pair_select(torch.from_numpy(rewards).cuda())
    pr = oracle.pair_select(rewards)["pair_rows"]
    tok = synth.tokens_rows(3, np.arange(P * K * T), 32000).reshape(P * K, T)
    mask = synth.mask_for(3, np.arange(P * K), T, "prefix", 11)
    ref = synth.rewards_for(4, P * K, 1).reshape(-1).astype(np.float32)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    t, m, r = odpo.gather_pairs(sel.pair_rows, torch.from_numpy(tok).cuda(),
                                torch.from_numpy(mask).cuda(), torch.from_numpy(ref).cuda(),
                                status=status)
    rows = pr.reshape(-1)
    assert np.array_equal(t.cpu().numpy(), tok[rows])
    assert np.array_equal(m.cpu().numpy(), mask[rows])
    assert np.array_equal(r.cpu().numpy(), ref[rows])
    assert int(status.item()) == 0
    bad = sel.pair_rows.clone()
    bad[5, 1] = P * K + 3
    t2, m2, _ = odpo.gather_pairs(bad, torch.from_numpy(tok).cuda(), torch.from_numpy(mask).cuda(),
                                  status=status)
    assert int(status.item()) & odpo.FLAGS["PAIR_RANGE"]
    assert torch.count_nonzero(t2[11]).item() == 0 and torch.count_nonzero(m2[11]).item() == 0


# ------------------------------------------------------------------ PSYNC at full Pythia size
@pytest.mark.parametrize("lag", [1, 4, 12])
def test_psync_full_pythia(odpo, lag):
    """The pair-synchronous split-V schedule at the BASELINE Pythia shape (the shape it is for),
    for several lags: deterministic, the same integer statistics and status as FUSED, sequence
    log-probs / z / loss within the bf16 contract of FUSED's (different row reduction trees),
    dlogits within one bf16 ulp of FUSED's, and sampled pairs against the oracle."""
    from synth.configs import CONFIGS
    w = CONFIGS["pythia"]
    b = Batch(w.P, w.T, w.V, w.dtype, seed=0, host=False)
    ref = torch.full((b.B,), -float(w.T) * 0.08, dtype=torch.float32, device="cuda")
    fused = run_loss(odpo, b, ref, w.beta, "fused")
    ps = run_loss(odpo, b, ref, w.beta, "psync", lag_pairs=lag)
    again = run_loss(odpo, b, ref, w.beta, "psync", lag_pairs=lag)
    assert torch.equal(ps.dlogits, again.dlogits) and torch.equal(ps.stats, again.stats)
    assert int(ps.status.item()) == int(fused.status.item()) == 0
    sf, sp = fused.stats.cpu().numpy(), ps.stats.cpu().numpy()
    for i in (0, 8, 9):
        assert sf[i] == sp[i]
    a_ = fused.seq_logp.cpu().double().numpy()
    b_ = ps.seq_logp.cpu().double().numpy()
    assert np.all(np.abs(a_ - b_) <= 2e-5 * np.maximum(np.abs(a_), 1.0))
    d = (ps.dlogits.float() - fused.dlogits.float()).abs()
    assert bool((d <= 2.0 ** -7 * fused.dlogits.float().abs() + 1e-12).all())
    pairs = synth.permutation(3, w.P)[:2]
    seqs = np.stack([2 * pairs, 2 * pairs + 1], 1).reshape(-1)
    o = oracle.online_dpo_loss_fwd_bwd(b.host_rows(seqs), np.full(len(seqs), -float(w.T) * 0.08, np.float32),
                                       b.tokens[seqs], b.mask[seqs], w.beta, p_global=w.P,
                                       n_threads=NCPU)
    check_seq(ps.seq_logp.cpu().numpy()[seqs], o["seq_logp"], w.dtype)


# ------------------------------------------------------------------------ split-row backward
@pytest.mark.parametrize("V,dt,pad", [(32767, "bf16", 0), (32768, "bf16", 0), (32769, "bf16", 0),
                                      (65552, "bf16", 0), (100000, "bf16", 0), (16384, "f32", 0),
                                      (16391, "f32", 0), (50304, "bf16", 8), (131072, "bf16", 0)])
def test_two_pass_piece_boundaries(odpo, V, dt, pad):
    """k_row_bwd_split cuts each row into one-batch pieces (S = ceil(vectors / (threads x 4)),
    32-byte vectors on 32-byte aligned rows, else 16-byte): around piece and vector boundaries,
    with the sampled token placed in the first, a middle and the last piece and in the ragged
    tail, the two-pass dlogits equal FUSED's (the engine's in-kernel backward, the same
    per-element arithmetic) bit for bit, and the oracle on every row.  pad: extra row elements
    (a row stride that is 16- but not 32-byte aligned for bf16 pad 8)."""
    P, T = 2, 4
    b = Batch(P, T, V, dt, seed=11, host=False)
    if pad:
        es = 4 if dt == "f32" else 2
        x = torch.empty((b.B, T, V + pad), dtype=b.d_logits.dtype, device="cuda")[:, :, :V]
        x.copy_(b.d_logits)
        b.d_logits = x
    tok = b.d_tokens.clone()
    places = [0, V // 3, V // 2 + 1, V - 1, V - 2, 17, (V // 16) * 16 - 1, V // 7]
    for i in range(b.B * T):
        tok.view(-1)[i] = places[i % len(places)] % V
    b.d_tokens = tok
    b.tokens = tok.cpu().numpy()
    ref = torch.full((b.B,), -3.0 * T, device="cuda")
    two = run_loss(odpo, b, ref, 0.1, "two_pass")
    fus = run_loss(odpo, b, ref, 0.1, "fused")
    assert torch.equal(two.dlogits, fus.dlogits)
    assert torch.equal(two.stats[:10], fus.stats[:10])
    assert int(two.status.item()) == 0
    h = Batch(P, T, V, dt, seed=11, host=True)
    h.tokens = b.tokens
    o = oracle.online_dpo_loss_fwd_bwd(h.h_logits if not pad else h.h_logits, ref.cpu().numpy(),
                                       b.tokens, h.mask, 0.1, want_dlogits=True, n_threads=NCPU)
    coef = coef_from_oracle(o, P, P, 0.1, 1.0, None, b.B)
    check_dlogits(to_f64(two.dlogits), o["dlogits"], coef[:, None, None], dt)
