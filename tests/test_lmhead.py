"""NEXT-2, forward part: sequence log-probs from the LM head without
materialising the logits.  CPU tests pin the oracle (closed form, brute force); GPU tests
compare the tcgen05 kernel (odpo_lmhead_seq_logprobs) with it element by element."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth


# ------------------------------------------------------------------ oracle pins (CPU)
def test_oracle_zero_head_is_uniform():
    """W = 0: every logit is 0, so log p = -log V and lse = log V exactly."""
    B, T, d, V = 2, 3, 64, 50
    h, _ = synth.lmhead_inputs(1, np.arange(B * T), d, V)
    w = np.zeros((V, d))
    tok = synth.tokens_rows(1, np.arange(B * T), V).reshape(B, T)
    mask = np.ones((B, T), np.uint8)
    o = oracle.lmhead_seq_logprobs(h.reshape(B, T, d), w, tok, mask)
    assert np.allclose(o["tok_logp"], -math.log(V), rtol=0, atol=1e-15)
    assert np.allclose(o["row_lse"], math.log(V), rtol=0, atol=1e-15)
    assert np.allclose(o["seq_logp"], -T * math.log(V), rtol=1e-15)


@pytest.mark.parametrize("invT", [1.0, 1 / 0.7])
def test_oracle_brute_force(invT):
    """Tiny shapes, pure-Python loops: logits[r, v] = sum_i h[r, i] w[v, i] (PAPER.md:83 with
    the LM head written out), log p = invT x_tok - log sum_v exp(invT x_v)."""
    B, T, d, V = 2, 3, 5, 7
    rows = np.arange(B * T)
    h, w = synth.lmhead_inputs(3, rows, d, V)
    tok = synth.tokens_rows(3, rows, V).reshape(B, T)
    mask = synth.mask_for(3, np.arange(B), T, "prefix", 2)
    o = oracle.lmhead_seq_logprobs(h.reshape(B, T, d), w, tok, mask, inv_temperature=invT)
    it = float(np.float32(invT))
    for b in range(B):
        S = 0.0
        for t in range(T):
            r = b * T + t
            x = [math.fsum(h[r, i] * w[v, i] for i in range(d)) for v in range(V)]
            mx = max(x)
            lse = it * mx + math.log(math.fsum(math.exp(it * (xv - mx)) for xv in x))
            lp = it * x[tok[b, t]] - lse
            if mask[b, t]:
                assert abs(o["tok_logp"][b, t] - lp) <= 1e-12
                S += lp
        assert abs(o["seq_logp"][b] - S) <= 1e-11


# ------------------------------------------------------------------ GPU parity

CASES = [
    # (B, T, d, V, mask, invT): ragged vocabulary tile, ragged row block, several raster groups
    (2, 5, 128, 1000, "dense", 1.0),
    (3, 50, 256, 4133, "prefix", 1 / 0.7),
    (4, 53, 2560, 50304, "dense", 1.0),   # the Pythia-2.8B LM head (d = 2560, V = 50304)
    (70, 64, 64, 300, "prefix", 1.0),     # 4480 rows = 35 row blocks: > 1 raster group of rows
    (2, 64, 4096, 128256, "prefix", 1.0), # the LLaMA-3.1-8B head; 128 rows: the CTA pair's
                                          # second half-block is all out of range
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"B{c[0]}T{c[1]}d{c[2]}V{c[3]}{c[4]}t{c[5]:.2f}")
@pytest.mark.gpu
@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")
def test_lmhead_parity(case):
    import paper_2410_18252_b200 as odpo
    B, T, d, V, mk, invT = case
    rows = np.arange(B * T)
    h, w = synth.lmhead_inputs(7, rows, d, V)
    tok = synth.tokens_rows(7, rows, V).reshape(B, T).astype(np.int32)
    mask = synth.mask_for(7, np.arange(B), T, mk, max(1, T // 2))
    hd = torch.from_numpy(h.reshape(B, T, d)).to(torch.bfloat16).cuda()   # exact (bf16 grid)
    wd = torch.from_numpy(w).to(torch.bfloat16).cuda()
    seq, tlp, lse, st = odpo.lmhead_seq_logprobs(hd, wd, torch.from_numpy(tok).cuda(),
                                                 torch.from_numpy(mask).cuda(), inv_temperature=invT)
    torch.cuda.synchronize()
    o = oracle.lmhead_seq_logprobs(h.reshape(B, T, d), w, tok, mask, inv_temperature=invT,
                                   n_threads=8)
    assert int(st.item()) == 0
    # fp32 tensor-core accumulation of exact bf16 products: per-token error << the bf16
    # contract (2e-3 relative on sequence log-probs)
    g = tlp.cpu().numpy().astype(np.float64)
    assert np.all(np.abs(g - o["tok_logp"]) <= 1e-4 * np.maximum(1.0, np.abs(o["tok_logp"])))
    gl = lse.cpu().numpy().astype(np.float64)
    m = mask == 1
    assert np.all(np.abs(gl[m] - o["row_lse"][m]) <= 1e-4 * np.maximum(1.0, np.abs(o["row_lse"][m])))
    S = seq.cpu().numpy().astype(np.float64)
    assert np.all(np.abs(S - o["seq_logp"]) <= 2e-3 * np.maximum(1.0, np.abs(o["seq_logp"])))
    assert np.all(np.abs(S - o["seq_logp"]) <= 1e-4 * np.maximum(1.0, np.abs(o["seq_logp"])))


@pytest.mark.gpu
@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")
def test_lmhead_token_range_flag():
    import paper_2410_18252_b200 as odpo
    B, T, d, V = 1, 4, 64, 300
    h, w = synth.lmhead_inputs(2, np.arange(B * T), d, V)
    tok = np.array([[0, 5, V, 7]], np.int32)
    mask = np.ones((B, T), np.uint8)
    _, _, _, st = odpo.lmhead_seq_logprobs(torch.from_numpy(h.reshape(B, T, d)).to(torch.bfloat16).cuda(),
                                           torch.from_numpy(w).to(torch.bfloat16).cuda(),
                                           torch.from_numpy(tok).cuda(), torch.from_numpy(mask).cuda())
    assert int(st.item()) & odpo.FLAGS["TOKEN_RANGE"]


@pytest.mark.parametrize("permute", [False, True])
@pytest.mark.gpu
@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")
def test_lmhead_dpo_loss_parity(permute):
    """The Online-DPO loss forward from the LM head (odpo_lmhead_seq_logprobs ->
    odpo_online_dpo_loss_from_token_logp) against the oracle's loss on the head's fp64 logits:
    sequence log-probs, z, loss and the statistics, and row_scale = coef_b * mask."""
    import paper_2410_18252_b200 as odpo
    P, T, d, V, extra = 5, 9, 128, 1000, (2 if permute else 0)
    B = 2 * P + extra
    rows = np.arange(B * T)
    h, w = synth.lmhead_inputs(11, rows, d, V)
    tok = synth.tokens_rows(11, rows, V).reshape(B, T).astype(np.int32)
    mask = synth.mask_for(11, np.arange(B), T, "prefix", 5)
    pr = synth.permutation(11, B)[: 2 * P].reshape(P, 2).astype(np.int32) if permute else None
    ref = (synth.rewards_for(11, B, 1).reshape(-1) - 40.0).astype(np.float32)
    beta = 0.1
    out = odpo.lmhead_online_dpo_loss_fwd(
        torch.from_numpy(h.reshape(B, T, d)).to(torch.bfloat16).cuda(),
        torch.from_numpy(w).to(torch.bfloat16).cuda(), torch.from_numpy(ref).cuda(),
        torch.from_numpy(tok).cuda(), torch.from_numpy(mask).cuda(), beta,
        pair_rows=None if pr is None else torch.from_numpy(pr).cuda(), p_global=P + 1)
    torch.cuda.synchronize()
    logits = (h @ w.T).reshape(B, T, V)
    o = oracle.online_dpo_loss_fwd_bwd(logits, ref, tok, mask, beta, pair_rows=pr, p_global=P + 1,
                                       unscaled=True, n_threads=8)
    live = np.arange(B) if pr is None else pr.reshape(-1)
    S = out.seq_logp.cpu().numpy().astype(np.float64)
    assert np.all(np.abs(S[live] - o["seq_logp"][live]) <= 1e-4 * np.maximum(1, np.abs(o["seq_logp"][live])))
    z = out.z.cpu().numpy().astype(np.float64)
    assert np.all(np.abs(z - o["z"]) <= 1e-4 * np.maximum(1, np.abs(o["z"])))
    from gpu_helpers import check_stats
    check_stats(out.stats.cpu().numpy(), o, "f32", beta, ref, pr, Pg=P + 1, tol=1e-4)
    rs = out.row_scale.cpu().numpy().astype(np.float64)
    assert np.all(np.abs(rs - o["row_scale"]) <= 1e-4 * np.abs(o["row_scale"]) + 1e-12)
    assert int(out.status.item()) & ~odpo.FLAGS["DEGENERATE_PAIR"] == 0


# ------------------------------------------------------------------ NEXT-2 backward
def _grad_case(seed=13, P=3, T=4, d=16, V=40, permute=True):
    B = 2 * P + (1 if permute else 0)
    rows = np.arange(B * T)
    h, w = synth.lmhead_inputs(seed, rows, d, V)
    tok = synth.tokens_rows(seed, rows, V).reshape(B, T).astype(np.int32)
    mask = synth.mask_for(seed, np.arange(B), T, "prefix", 3)
    pr = synth.permutation(seed, B)[: 2 * P].reshape(P, 2).astype(np.int32) if permute else None
    ref = (synth.rewards_for(seed, B, 1).reshape(-1) - 12.0).astype(np.float32)
    return B, T, d, V, h.reshape(B, T, d), w, tok, mask, pr, ref


def test_oracle_grad_central_differences():
    """dL/dhidden and dL/dweight of the oracle loss (fp64 logits = hidden @ weight.T) by central
    differences: pins the chain rule (a dropped row_scale, a transposed product or a wrong
    sign fails it)."""
    B, T, d, V, h, w, tok, mask, pr, ref = _grad_case()
    beta, eps = 0.5, 1e-5
    g = oracle.lmhead_dpo_grad(h, w, ref, tok, mask, beta, pair_rows=pr)

    def loss(hh, ww):
        lg = np.ascontiguousarray((hh.reshape(B * T, d) @ ww.T).reshape(B, T, V))
        return oracle.online_dpo_loss_fwd_bwd(lg, ref, tok, mask, beta, pair_rows=pr)["stats"][1]

    rng = np.random.default_rng(0)
    for _ in range(6):
        b, t, i = rng.integers(B), rng.integers(T), rng.integers(d)
        hp, hm = h.copy(), h.copy()
        hp[b, t, i] += eps
        hm[b, t, i] -= eps
        fd = (loss(hp, w) - loss(hm, w)) / (2 * eps)
        assert abs(fd - g["dhidden"][b, t, i]) <= 1e-6 + 1e-5 * abs(fd), (b, t, i, fd, g["dhidden"][b, t, i])
        v, j = rng.integers(V), rng.integers(d)
        wp, wm = w.copy(), w.copy()
        wp[v, j] += eps
        wm[v, j] -= eps
        fd = (loss(h, wp) - loss(h, wm)) / (2 * eps)
        assert abs(fd - g["dweight"][v, j]) <= 1e-6 + 1e-5 * abs(fd), (v, j, fd, g["dweight"][v, j])
    assert np.any(g["dhidden"] != 0) and np.any(g["dweight"] != 0)


@pytest.mark.parametrize("shape", [(5, 9, 128, 1000, 256, 1.0), (40, 53, 256, 4133, 1024, 1.0),
                                   (6, 11, 192, 3001, 256, 1 / 0.7), (3, 200, 640, 2500, 512, 1.0)],
                         ids=lambda s: f"P{s[0]}T{s[1]}d{s[2]}V{s[3]}c{s[4]}t{s[5]:.2f}")
@pytest.mark.gpu
@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")
def test_lmhead_grad_parity(shape):
    """odpo_lmhead_grad (logits recomputed on tcgen05 chunk by chunk, G and G^T in bf16, the
    library's tcgen05 GEMMs) against the oracle's chain rule, with row_lse / row_scale from the
    GPU forward, ELEMENT BY ELEMENT: dhidden[r, i] = sum_v G[r, v] W[v, i] carries G's bf16
    rounding (2^-9 relative per term) and the fp32 accumulation, so each element is held to
    2^-8 (|G| |W|)[r, i] (the sum of the magnitudes of its terms; G sums to ~0 over v, so a
    bound relative to |dhidden| itself would not be rigorous), likewise dweight with |G|^T |H|."""
    import paper_2410_18252_b200 as odpo
    P, T, d, V, chunk, invT = shape
    B, _, _, _, h, w, tok, mask, pr, ref = _grad_case(seed=17, P=P, T=T, d=d, V=V)
    beta = 0.1
    hd = torch.from_numpy(h).to(torch.bfloat16).cuda()
    wd = torch.from_numpy(w).to(torch.bfloat16).cuda()
    td, md = torch.from_numpy(tok).cuda(), torch.from_numpy(mask).cuda()
    prd = torch.from_numpy(pr).cuda()
    out = odpo.lmhead_online_dpo_loss_fwd(hd, wd, torch.from_numpy(ref).cuda(), td, md, beta,
                                          pair_rows=prd, inv_temperature=invT)
    dh, dw = odpo.lmhead_grad(hd, wd, td, out.row_lse, out.row_scale, inv_temperature=invT,
                              chunk_rows=chunk)
    torch.cuda.synchronize()
    o = oracle.lmhead_dpo_grad(h, w, ref, tok, mask, beta, pair_rows=pr, inv_temperature=invT,
                               n_threads=8)
    aG = np.abs(o["G"])
    mag_h = (aG @ np.abs(w)).reshape(B, T, d)
    mag_w = aG.T @ np.abs(h.reshape(B * T, d))
    for gpu, orc, mag in ((dh.cpu().double().numpy(), o["dhidden"], mag_h),
                          (dw.cpu().double().numpy(), o["dweight"], mag_w)):
        err = np.abs(gpu - orc)
        bound = 2.0 ** -8 * mag + 1e-12
        assert np.all(err <= bound), (float(np.max(err - bound)), float(np.max(err / np.maximum(mag, 1e-30))))
        assert np.linalg.norm(gpu - orc) <= 1e-2 * np.linalg.norm(orc)


# ------------------------------------------------------------------ NEXT-2 chunked learner step
@pytest.mark.parametrize("shape", [(3, 9, 128, 1000, 1), (3, 9, 128, 1000, 2), (4, 53, 256, 4133, 3),
                                   (2, 64, 640, 2500, 5), (3, 16, 128, 12345, 2)],
                         ids=lambda s: f"P{s[0]}T{s[1]}d{s[2]}V{s[3]}cp{s[4]}")
@pytest.mark.gpu
@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")
def test_lmhead_dpo_step_parity(shape):
    """odpo_lmhead_dpo_step (per chunk of pairs: bf16 logits and per-tile (m, log1p r, x_tok)
    partials from the library's head kernel, the loss merged from the partials with dlogits in
    place, dhidden / dweight from the library GEMMs; V = 12345 has 49 tiles, the warp-per-row
    merge) against the oracle on the same bf16
    logits: the head's products are dyadic (synth.lmhead_inputs), so the fp32 tensor-core sum is
    exact and both sides round the same value to bf16.  Sequence log-probs, z and all ten
    statistics at the bf16 contract; dhidden / dweight element-wise within the propagated R17
    bound of the dlogits: 2^-7 (|G| |W|) + 2^-20 |coef| sum|W| (resp. with |H|)."""
    import paper_2410_18252_b200 as odpo
    from gpu_helpers import check_seq, check_stats
    P, T, d, V, cp = shape
    B = 2 * P
    rows = np.arange(B * T)
    h, w = synth.lmhead_inputs(19, rows, d, V)
    tok = synth.tokens_rows(19, rows, V).reshape(B, T).astype(np.int32)
    mask = synth.mask_for(19, np.arange(B), T, "prefix", max(2, T // 2))
    logits = (h @ w.T).reshape(B, T, V)
    bits = oracle.to_bf16_bits(logits.astype(np.float32))
    S0 = oracle.seq_logprobs(bits, tok, mask)["seq_logp"]
    ref = (S0 + np.where(np.arange(B) % 2 == 0, 0.5, -0.25)).astype(np.float32)
    beta, Pg = 0.1, P + 2
    out, dh, dw = odpo.lmhead_dpo_step(
        torch.from_numpy(h.reshape(B, T, d)).to(torch.bfloat16).cuda(),
        torch.from_numpy(w).to(torch.bfloat16).cuda(), torch.from_numpy(ref).cuda(),
        torch.from_numpy(tok).cuda(), torch.from_numpy(mask).cuda(), beta, p_global=Pg,
        chunk_pairs=cp)
    torch.cuda.synchronize()
    o = oracle.online_dpo_loss_fwd_bwd(bits, ref, tok, mask, beta, p_global=Pg, want_dlogits=True)
    assert int(out.status.item()) == 0
    check_seq(out.seq_logp.cpu().numpy(), o["seq_logp"], "bf16")
    check_stats(out.stats.cpu().numpy(), o, "bf16", beta, ref, None, Pg=Pg)
    G = o["dlogits"].reshape(B * T, V)
    aG = np.abs(G)
    cabs = np.zeros(B * T)
    for p in range(P):
        sig = 1.0 / (1.0 + np.exp(o["z"][p]))
        c = float(np.float32(beta)) * sig / Pg
        cabs[(2 * p) * T:(2 * p + 2) * T] = c
    dh_o = (G @ w).reshape(B, T, d)
    dw_o = G.T @ h.reshape(B * T, d)
    bh = 2.0 ** -7 * (aG @ np.abs(w)) + 2.0 ** -20 * cabs[:, None] * np.abs(w).sum(0)[None, :]
    bw = 2.0 ** -7 * (aG.T @ np.abs(h.reshape(B * T, d))) + \
        2.0 ** -20 * (cabs[:, None] * np.abs(h.reshape(B * T, d))).sum(0)[None, :]
    eh = np.abs(dh.cpu().double().numpy().reshape(B * T, d) - dh_o.reshape(B * T, d))
    ew = np.abs(dw.cpu().double().numpy() - dw_o)
    assert np.all(eh <= bh + 1e-12), float(np.max(eh - bh))
    assert np.all(ew <= bw + 1e-12), float(np.max(ew - bw))


@pytest.mark.gpu
@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")
def test_lmhead_dynamic_tile_order_sampled():
    """A head large enough for the CTA-pair kernel's dynamic tile order (>= 512 tiles per pair:
    32768 rows = 128 pair-blocks x 296 vocabulary tiles = 37888 tiles over 74 pairs): every
    tile's partial lands in its fixed slot whatever pair claims it, so sampled rows match the
    oracle (the head's fp64 matmul, then seq_logprobs) at the usual 1e-4 bound, and two calls
    give the same bits."""
    import paper_2410_18252_b200 as odpo
    B, T, d, V = 32, 1024, 64, 75776
    rows = np.arange(B * T)
    h, w = synth.lmhead_inputs(23, rows, d, V)
    tok = synth.tokens_rows(23, rows, V).reshape(B, T).astype(np.int32)
    mask = np.ones((B, T), np.uint8)
    hd = torch.from_numpy(h.reshape(B, T, d)).to(torch.bfloat16).cuda()
    wd = torch.from_numpy(w).to(torch.bfloat16).cuda()
    tk, mk = torch.from_numpy(tok).cuda(), torch.from_numpy(mask).cuda()
    seq, tlp, lse, st = odpo.lmhead_seq_logprobs(hd, wd, tk, mk)
    seq2, tlp2, lse2, _ = odpo.lmhead_seq_logprobs(hd, wd, tk, mk)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    assert torch.equal(tlp, tlp2) and torch.equal(lse, lse2) and torch.equal(seq, seq2)
    take = np.unique(np.concatenate([np.arange(0, B * T, 997), [1, 255, 256, 4095, B * T - 1]]))
    o = oracle.lmhead_seq_logprobs(h[take].reshape(1, len(take), d), w,
                                   tok.reshape(-1)[take].reshape(1, -1),
                                   np.ones((1, len(take)), np.uint8), n_threads=8)
    g = tlp.reshape(-1).cpu().numpy().astype(np.float64)[take]
    assert np.all(np.abs(g - o["tok_logp"].reshape(-1)) <= 1e-4 * np.maximum(1.0, np.abs(o["tok_logp"].reshape(-1))))
    gl = lse.reshape(-1).cpu().numpy().astype(np.float64)[take]
    assert np.all(np.abs(gl - o["row_lse"].reshape(-1)) <= 1e-4 * np.maximum(1.0, np.abs(o["row_lse"].reshape(-1))))
