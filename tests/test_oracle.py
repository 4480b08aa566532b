"""Pins for the CPU oracle (no GPU).  Each test checks the oracle against something
other than itself: printed worked examples (tests/golden/), closed forms,
brute force in 50-digit decimal arithmetic, a library routine (scipy), finite
differences, and invariants fixed by the mathematics (SURVEY.md §8(c) test matrix
O-1..O-10)."""
import itertools
import math
import struct
from decimal import Decimal, getcontext

import numpy as np
import pytest

from helpers import golden_rows

pytestmark = pytest.mark.filterwarnings("ignore::RuntimeWarning")


def f32_hex(x):
    return struct.pack(">f", np.float32(x)).hex()


# ----------------------------------------------------------------- O-1 / O-2 pair_select
def test_pair_select_spec_vectors(orc):
    """SPEC.md:191-192, 383, 392-394 worked examples (golden file)."""
    for rw, ch, rj, mhex, deg in golden_rows("spec_pair_select.txt"):
        r = np.array([[float(v) for v in rw.split(",")]], dtype=np.float32)
        out = orc.pair_select(r)
        assert out["chosen"][0] == int(ch), rw
        assert out["rejected"][0] == int(rj), rw
        assert f32_hex(out["margin"][0]) == mhex, rw
        assert bool(out["status"] & orc.FLAG_DEGENERATE_PAIR) == bool(int(deg)), rw
        assert out["sel_stats"][1] == float(int(deg))


@pytest.mark.parametrize("K", [2, 3, 4])
def test_pair_select_exhaustive(orc, K):
    """Brute force over all K-tuples from {-1, 0, 0.5, 1}: first max / last min,
    r[chosen] >= r[i] >= r[rejected], degenerate iff max == min."""
    vals = [-1.0, 0.0, 0.5, 1.0]
    groups = np.array(list(itertools.product(vals, repeat=K)), dtype=np.float32)
    out = orc.pair_select(groups)
    for p, g in enumerate(groups.tolist()):
        mx, mn = max(g), min(g)
        exp_c = g.index(mx)
        exp_r = K - 1 - g[::-1].index(mn)
        assert out["chosen"][p] == exp_c and out["rejected"][p] == exp_r, g
        assert all(g[out["chosen"][p]] >= v >= g[out["rejected"][p]] for v in g)
        assert tuple(out["pair_rows"][p]) == (p * K + exp_c, p * K + exp_r)
        assert out["margin"][p] == np.float32(np.float32(mx) - np.float32(mn))
    ndeg = sum(1 for g in groups.tolist() if max(g) == min(g))
    assert out["sel_stats"][1] == ndeg
    # antisymmetry at K = 2: swapping two distinct scores swaps chosen/rejected
    if K == 2:
        sw = groups[:, ::-1].copy()
        o2 = orc.pair_select(sw)
        distinct = groups[:, 0] != groups[:, 1]
        assert np.all(o2["chosen"][distinct] == out["rejected"][distinct])
        assert np.all(o2["rejected"][distinct] == out["chosen"][distinct])


def test_pair_select_eos_penalty_replaces(orc):
    """PAPER.md:434-435 / 518-519: the penalty VALUE replaces the score (reading R7)."""
    r = np.array([[0.4, 0.2], [0.4, 0.2], [-3.0, 5.0]], dtype=np.float32)
    e = np.array([[1, 1], [0, 1], [1, 0]], dtype=np.uint8)
    out = orc.pair_select(r, e, eos_penalty=-10.0)
    assert list(out["chosen"]) == [0, 1, 0]
    assert list(out["rejected"]) == [1, 0, 1]
    assert out["margin"][1] == np.float32(np.float32(0.2) - np.float32(-10.0))
    assert out["sel_stats"][2] == 2.0  # two truncated completions
    out = orc.pair_select(np.array([[np.nan, 1.0]], np.float32))
    assert out["status"] & orc.FLAG_NONFINITE_REWARD


# --------------------------------------------------------------------- O-3 LSE brute force
def _decimal_logsoftmax(row, tok, invT):
    getcontext().prec = 50
    ys = [Decimal(float(v)) * Decimal(float(np.float32(invT))) for v in row]
    lse = sum((y.exp() for y in ys), Decimal(0)).ln()   # no max shift
    return float(ys[tok] - lse), float(lse)


@pytest.mark.parametrize("V", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("dist", ["grid", "normal"])
def test_lse_bruteforce_decimal(orc, V, dist):
    rng = np.random.default_rng(V * 7 + (dist == "normal"))
    B, T = 10, 20
    if dist == "grid":
        x = rng.integers(-256, 256, size=(B, T, V)).astype(np.float64) / 64.0
    else:
        x = rng.normal(0.0, 10.0, size=(B, T, V))
    tok = rng.integers(0, V, size=(B, T)).astype(np.int32)
    mask = np.ones((B, T), np.uint8)
    for invT in (1.0, 1 / 0.7):
        out = orc.seq_logprobs(x, tok, mask, inv_temperature=invT)
        for b in range(B):
            for t in range(T):
                lp, lse = _decimal_logsoftmax(x[b, t], tok[b, t], invT)
                # a few double ulps of the largest intermediate (|lse|, |y|)
                scale = max(1.0, abs(lse), float(np.max(np.abs(x[b, t]))) * invT)
                assert abs(out["tok_logp"][b, t] - lp) <= 4.5e-16 * 4 * scale
                assert abs(out["row_lse"][b, t] - lse) <= 4.5e-16 * 4 * scale
            assert abs(out["seq_logp"][b] - out["tok_logp"][b].sum()) <= 1e-13 * max(
                1.0, abs(out["seq_logp"][b]))


def test_v1_and_v2_closed_forms(orc):
    x1 = np.array([[[3.5], [-7.0]]])
    out = orc.seq_logprobs(x1, np.zeros((1, 2), np.int32), np.ones((1, 2), np.uint8))
    assert np.all(out["tok_logp"] == 0.0) and out["seq_logp"][0] == 0.0
    rng = np.random.default_rng(2)
    x2 = rng.normal(0, 3, size=(3, 4, 2))
    tok = rng.integers(0, 2, size=(3, 4)).astype(np.int32)
    out = orc.seq_logprobs(x2, tok, np.ones((3, 4), np.uint8))
    for b in range(3):
        for t in range(4):
            k = tok[b, t]
            expect = -math.log1p(math.exp(x2[b, t, 1 - k] - x2[b, t, k]))
            assert abs(out["tok_logp"][b, t] - expect) < 1e-15


def test_scipy_logsumexp_large_rows(orc):
    """Library routine pin at a realistic vocabulary size (scipy.special.logsumexp)."""
    from scipy.special import logsumexp
    rng = np.random.default_rng(5)
    B, T, V = 2, 3, 50304
    x = (rng.integers(-128, 128, size=(B, T, V)) / 64.0).astype(np.float32)
    tok = rng.integers(0, V, size=(B, T)).astype(np.int32)
    x[0, :, :][np.arange(T), tok[0]] = 14.0
    out = orc.seq_logprobs(x, tok, np.ones((B, T), np.uint8))
    for b in range(B):
        for t in range(T):
            ref = float(x[b, t, tok[b, t]]) - logsumexp(x[b, t].astype(np.float64))
            # recursive-summation error bound of the oracle's sequential sum: V * 2^-53
            assert abs(out["tok_logp"][b, t] - ref) <= V * 2.0 ** -53


# -------------------------------------------------------------------------- O-4 uniform
@pytest.mark.parametrize("V", [7, 50304])
def test_uniform_rows(orc, V):
    """uniform logits -> S = -L ln V."""
    B, T = 3, 5
    x = np.full((B, T, V), 1.25, dtype=np.float32)
    tok = (np.arange(B * T).reshape(B, T) * 31 % V).astype(np.int32)
    mask = np.zeros((B, T), np.uint8)
    L = [1, 3, 5]
    for b in range(B):
        mask[b, :L[b]] = 1
    out = orc.seq_logprobs(x, tok, mask)
    for b in range(B):
        exp_ = -L[b] * math.log(V)
        assert abs(out["seq_logp"][b] - exp_) <= 1e-14 * abs(exp_)


def test_shift_invariance_and_additivity(orc):
    rng = np.random.default_rng(11)
    B, T, V = 2, 6, 13
    x = rng.normal(size=(B, T, V))
    tok = rng.integers(0, V, size=(B, T)).astype(np.int32)
    mask = np.ones((B, T), np.uint8)
    a = orc.seq_logprobs(x, tok, mask)
    b_ = orc.seq_logprobs(x + 3.25, tok, mask)
    assert np.max(np.abs(a["tok_logp"] - b_["tok_logp"])) < 1e-13
    # additivity: masking token (0, 2) removes exactly its term
    m2 = mask.copy()
    m2[0, 2] = 0
    c = orc.seq_logprobs(x, tok, m2)
    assert abs((a["seq_logp"][0] - c["seq_logp"][0]) - a["tok_logp"][0, 2]) < 1e-13
    assert c["seq_logp"][1] == a["seq_logp"][1]


def test_bf16_decode_and_strides(orc):
    """bf16 bit patterns decode exactly; strided views equal contiguous inputs."""
    rng = np.random.default_rng(3)
    x = (rng.integers(-128, 128, size=(2, 7, 40)) / 64.0).astype(np.float32)
    tok = rng.integers(0, 40, size=(2, 4)).astype(np.int32)
    mask = np.ones((2, 4), np.uint8)
    bits = orc.to_bf16_bits(x)
    assert np.array_equal(orc.bf16_bits_to_f64(bits), x.astype(np.float64))
    a = orc.seq_logprobs(np.ascontiguousarray(x[:, 2:6]), tok, mask)
    b_ = orc.seq_logprobs(bits[:, 2:6], tok, mask)
    assert np.array_equal(a["seq_logp"], b_["seq_logp"])


def test_thread_count_invariance(orc):
    rng = np.random.default_rng(4)
    B, T, V = 8, 5, 33
    x = rng.normal(size=(B, T, V)).astype(np.float32)
    tok = rng.integers(0, V, size=(B, T)).astype(np.int32)
    mask = (rng.random((B, T)) < 0.8).astype(np.uint8)
    mask[:, 0] = 1
    ref = rng.normal(-5, 1, size=B).astype(np.float32)
    a = orc.online_dpo_loss_fwd_bwd(x, ref, tok, mask, 0.1, want_dlogits=True, n_threads=1)
    b_ = orc.online_dpo_loss_fwd_bwd(x, ref, tok, mask, 0.1, want_dlogits=True, n_threads=5)
    for k in ("seq_logp", "z", "stats", "dlogits"):
        assert np.array_equal(a[k], b_[k]), k


# ------------------------------------------------------------------------ O-5 W1 golden
def test_w1_golden(orc):
    ln3 = math.log(3.0)
    x = np.array([[[ln3, 0.0]], [[0.0, ln3]]])
    tok = np.zeros((2, 1), np.int32)
    mask = np.ones((2, 1), np.uint8)
    ref = np.full(2, np.float32(math.log(0.5)), np.float32)
    for beta, Sc, Sr, z, loss, c0, c1, r0, r1 in golden_rows("w1_dpo.txt"):
        beta = float(beta)
        # ref_c == ref_r, so they cancel exactly in z; pass the fp32 value on both sides
        out = orc.online_dpo_loss_fwd_bwd(x, ref, tok, mask, beta, want_dlogits=True)
        assert abs(out["seq_logp"][0] - float(Sc)) < 1e-14
        assert abs(out["seq_logp"][1] - float(Sr)) < 1e-14
        zb = float(np.float32(beta)) * ln3  # beta enters as fp32
        assert abs(out["z"][0] - float(z) * (zb / (beta * ln3))) < 1e-14
        exp_loss = math.log1p(3.0 ** -float(np.float32(beta)))
        assert abs(out["stats"][1] - exp_loss) < 1e-14
        if beta == 1.0:
            assert abs(out["stats"][1] - float(loss)) < 1e-14
            g = out["dlogits"]
            assert np.allclose(g[0, 0], [float(c0), float(c1)], rtol=0, atol=1e-15)
            assert np.allclose(g[1, 0], [float(r0), float(r1)], rtol=0, atol=1e-15)
        else:
            g = out["dlogits"]
            scale = float(np.float32(beta)) / beta
            assert np.allclose(g[0, 0], [float(c0), float(c1)], rtol=2e-7 * max(1, scale), atol=0)
            assert np.allclose(g[1, 0], [float(r0), float(r1)], rtol=2e-7, atol=0)
            assert abs(out["stats"][1] - float(loss)) < 1e-8


def test_w1_golden_statistics(orc):
    """All ten loss statistics of the W1 worked example and of its swap, against the closed
    form (tests/golden/w1_stats.txt): the implicit-reward margin sum z, the chosen / rejected
    implicit rewards beta (S - ref), the sequence log-prob sums and the token counts."""
    ln3 = math.log(3.0)
    x = np.array([[[ln3, 0.0]], [[0.0, ln3]]])
    tok = np.zeros((2, 1), np.int32)
    mask = np.ones((2, 1), np.uint8)
    ref = np.full(2, np.float32(math.log(0.5)), np.float32)
    for case, beta, *vals in golden_rows("w1_stats.txt"):
        beta = float(beta)
        pr = np.array([[0, 1]] if case == "w1" else [[1, 0]], np.int32)
        out = orc.online_dpo_loss_fwd_bwd(x, ref, tok, mask, beta, pair_rows=pr)
        st = out["stats"]
        exp = [float(v) for v in vals]
        scale = float(np.float32(beta)) / beta  # beta enters as fp32
        assert st[0] == exp[0] and st[2] == exp[2] and st[8] == exp[8] and st[9] == exp[9]
        sgn = 1.0 if case == "w1" else -1.0
        assert abs(st[1] - math.log1p(3.0 ** (-sgn * float(np.float32(beta))))) < 1e-14
        assert abs(st[1] - exp[1]) < 1e-8 * max(1.0, abs(scale - 1) * 1e8)
        for i in (3, 4, 5):      # beta-linear columns
            assert abs(st[i] - exp[i] * scale) < 3e-9, (case, beta, i, st[i], exp[i])
        for i in (6, 7):
            assert abs(st[i] - exp[i]) < 1e-14, (case, beta, i)


def test_statistics_identities_and_swap(orc):
    """Identities the mathematics fixes for the margin statistics on a random batch:
    z_sum = r_chosen - r_rejected, r_chosen = beta (S_c_sum - ref_c_sum), S sums equal the
    per-sequence log-probs summed over chosen / rejected members, and swapping y+/y- of every
    pair exchanges the chosen and rejected columns and negates z_sum."""
    P = 300
    x, tok, mask, rng = _random_batch(21, P=P, T=4, V=7)
    ref = rng.normal(-5, 2, size=2 * P).astype(np.float32)
    pr = synth_perm_pairs(P, seed=4)
    beta = 0.25
    a = orc.online_dpo_loss_fwd_bwd(x, ref, tok, mask, beta, pair_rows=pr)
    b_ = orc.online_dpo_loss_fwd_bwd(x, ref, tok, mask, beta, pair_rows=pr[:, ::-1].copy())
    S = a["seq_logp"]
    c, r = pr[:, 0], pr[:, 1]
    sa = a["stats"]
    assert abs(sa[6] - S[c].sum()) < 1e-10 and abs(sa[7] - S[r].sum()) < 1e-10
    assert abs(sa[4] - beta * (S[c] - ref[c].astype(np.float64)).sum()) < 1e-10
    assert abs(sa[5] - beta * (S[r] - ref[r].astype(np.float64)).sum()) < 1e-10
    assert abs(sa[3] - (sa[4] - sa[5])) < 1e-10
    assert sa[8] == mask[c].sum() and sa[9] == mask[r].sum()
    sb = b_["stats"]
    assert sb[3] == -sa[3] or abs(sb[3] + sa[3]) < 1e-12
    for i, j in ((4, 5), (6, 7), (8, 9)):
        assert abs(sb[i] - sa[j]) < 1e-12 and abs(sb[j] - sa[i]) < 1e-12
    assert sa[2] + sb[2] == np.count_nonzero(a["z"])


def synth_perm_pairs(P, seed):
    """A random pairing of 2P rows (every row in exactly one pair)."""
    perm = np.random.default_rng(seed).permutation(2 * P).astype(np.int32)
    return perm.reshape(P, 2)


# ------------------------------------------------------------------ KL proxy (PPL)
@pytest.mark.parametrize("V", [1, 2, 7, 50304])
def test_ppl_uniform_rows_is_V(orc, V):
    """PAPER.md:121/333 KL proxy: on uniform rows every token has probability 1/V, so the
    perplexity of every completion is exactly V (closed form), whatever its length."""
    B, T = 3, 5
    x = np.full((B, T, V), 0.375, np.float32)
    tok = (np.arange(B * T).reshape(B, T) % V).astype(np.int32)
    mask = np.ones((B, T), np.uint8)
    mask[1, 2:] = 0
    mask[2, :] = 0
    o = orc.seq_ppl(x, tok, mask)
    assert abs(o["ppl"][0] - V) <= 1e-12 * V and abs(o["ppl"][1] - V) <= 1e-12 * V
    assert o["ppl"][2] == 1.0 and o["status"] & orc.FLAG_EMPTY_SEQ
    ps = o["ppl_stats"]
    assert ps[0] == 2 and abs(ps[1] - 2 * V) <= 1e-12 * V and ps[3] == T + 2
    assert abs(math.exp(-ps[2] / ps[3]) - V) <= 1e-12 * V


def test_ppl_two_token_closed_form(orc):
    """V = 2 rows x = (ln 3, 0) with token 0: p = 3/4 per token, so PPL = 4/3 for any length;
    mixing one p = 1/4 token into a length-2 completion gives PPL = (3/4 * 1/4)^(-1/2)."""
    ln3 = math.log(3.0)
    x = np.array([[[ln3, 0.0], [ln3, 0.0]], [[ln3, 0.0], [0.0, ln3]]])
    tok = np.zeros((2, 2), np.int32)
    o = orc.seq_ppl(x, tok, np.ones((2, 2), np.uint8))
    assert abs(o["ppl"][0] - 4.0 / 3.0) < 1e-14
    assert abs(o["ppl"][1] - (3.0 / 16.0) ** -0.5) < 1e-14


# ---------------------------------------------------------------------- O-6 ln 2 / O-7 swap
def _random_batch(seed, P=40, T=6, V=17, dtype=np.float64):
    rng = np.random.default_rng(seed)
    B = 2 * P
    x = rng.normal(0, 2, size=(B, T, V)).astype(dtype)
    tok = rng.integers(0, V, size=(B, T)).astype(np.int32)
    mask = (rng.random((B, T)) < 0.7).astype(np.uint8)
    mask[:, 0] = 1
    return x, tok, mask, rng


def test_ln2_when_policy_equals_reference(orc):
    """theta = init -> z = 0, loss = ln 2, coef = +-beta/(2P)."""
    P = 1000
    # exact ln 2 when ref carries S exactly: use f64 logits whose S is representable
    x2 = np.zeros((2 * P, 1, 4))
    tok2 = np.zeros((2 * P, 1), np.int32)
    m2 = np.ones((2 * P, 1), np.uint8)
    ref2 = np.full(2 * P, np.float32(-math.log(4.0)), np.float32)
    S2 = orc.seq_logprobs(x2, tok2, m2)["seq_logp"]
    out2 = orc.online_dpo_loss_fwd_bwd(x2, ref2, tok2, m2, 0.1, want_dlogits=True)
    assert np.all(S2 == S2[0])
    z = out2["z"]
    assert np.all(z == z[0]) and np.all(z == 0.0)
    assert abs(out2["stats"][1] - math.log(2.0)) < 1e-12  # SPEC.md:599 (1000 pairs, 1e-12)
    assert out2["stats"][2] == 0.0
    beta = float(np.float32(0.1))
    g = out2["dlogits"]
    # coef_c = beta * sigma(0) / P = beta / (2P); softmax = 1/4 uniform
    exp_c = beta / (2 * P)
    assert np.allclose(g[0, 0], exp_c * np.array([0.25 - 1, 0.25, 0.25, 0.25]), rtol=1e-15, atol=0)
    assert np.allclose(g[1, 0], -exp_c * np.array([0.25 - 1, 0.25, 0.25, 0.25]), rtol=1e-15, atol=0)


def test_swap_negates_z(orc):
    """swapping y+/y- maps z -> -z exactly; loss(swap) - loss = z."""
    P = 1000
    x, tok, mask, rng = _random_batch(2, P=P, T=3, V=5)
    ref = rng.normal(-4, 1, size=2 * P).astype(np.float32)
    pr = np.stack([np.arange(0, 2 * P, 2), np.arange(1, 2 * P, 2)], axis=1).astype(np.int32)
    a = orc.online_dpo_loss_fwd_bwd(x, ref, tok, mask, 0.05, pair_rows=pr)
    b_ = orc.online_dpo_loss_fwd_bwd(x, ref, tok, mask, 0.05, pair_rows=pr[:, ::-1].copy())
    assert np.array_equal(b_["z"], -a["z"])
    # per-pair: softplus(z) - softplus(-z) = z  -> summed over pairs / P
    assert abs((b_["stats"][1] - a["stats"][1]) * P - a["z"].sum()) < 1e-9
    assert b_["stats"][2] + a["stats"][2] == np.count_nonzero(a["z"])


# --------------------------------------------------------------------- O-8 finite differences
@pytest.mark.parametrize("beta", [0.03, 1.0])
@pytest.mark.parametrize("invT", [1.0, 1 / 0.7])
def test_gradient_finite_differences(orc, beta, invT):
    rng = np.random.default_rng(int(beta * 100) + int(invT * 10))
    B, T, V = 4, 3, 5
    x = rng.normal(0, 1.5, size=(B, T, V))
    tok = rng.integers(0, V, size=(B, T)).astype(np.int32)
    mask = (rng.random((B, T)) < 0.7).astype(np.uint8)
    mask[:, 0] = 1
    mask[1, 2] = 0
    ref = rng.normal(-3, 1, size=B).astype(np.float32)
    pr = np.array([[2, 1], [0, 3]], np.int32)
    Pg = 5
    base = orc.online_dpo_loss_fwd_bwd(x, ref, tok, mask, beta, pair_rows=pr, p_global=Pg,
                                       inv_temperature=invT, want_dlogits=True)
    g = base["dlogits"]
    h = 1e-6
    worst = 0.0
    for b in range(B):
        for t in range(T):
            for v in range(V):
                xp = x.copy()
                xp[b, t, v] += h
                xm = x.copy()
                xm[b, t, v] -= h
                lp = orc.online_dpo_loss_fwd_bwd(xp, ref, tok, mask, beta, pair_rows=pr, p_global=Pg,
                                                 inv_temperature=invT)["stats"][1]
                lm = orc.online_dpo_loss_fwd_bwd(xm, ref, tok, mask, beta, pair_rows=pr, p_global=Pg,
                                                 inv_temperature=invT)["stats"][1]
                fd = (lp - lm) / (2 * h)
                worst = max(worst, abs(fd - g[b, t, v]))
    assert worst <= 1e-8, worst
    # masked row is exactly zero
    assert np.all(g[1, 2] == 0.0)


# ------------------------------------------------------- O-8b factored (unscaled) gradient
def test_unscaled_factorisation_finite_differences(orc):
    """row_scale * G is the loss gradient (central differences, as O-8), G is the plain
    softmax - onehot of invT x (scipy), and masked / unreferenced rows are 0 in both."""
    from scipy.special import softmax
    rng = np.random.default_rng(11)
    B, T, V, invT, beta = 6, 3, 5, 1 / 0.7, 0.3
    x = rng.normal(0, 1.5, size=(B, T, V))
    tok = rng.integers(0, V, size=(B, T)).astype(np.int32)
    mask = np.ones((B, T), np.uint8)
    mask[1, 2] = 0
    ref = rng.normal(-3, 1, size=B).astype(np.float32)
    pr = np.array([[2, 1], [0, 3]], np.int32)   # rows 4, 5 unreferenced
    Pg = 3
    u = orc.online_dpo_loss_fwd_bwd(x, ref, tok, mask, beta, pair_rows=pr, p_global=Pg,
                                    inv_temperature=invT, want_dlogits=True, unscaled=True)
    G, rs = u["dlogits"], u["row_scale"]
    h = 1e-6
    worst = 0.0
    for b in range(4):
        for t in range(T):
            for v in range(V):
                xp = x.copy()
                xp[b, t, v] += h
                xm = x.copy()
                xm[b, t, v] -= h
                lp = orc.online_dpo_loss_fwd_bwd(xp, ref, tok, mask, beta, pair_rows=pr,
                                                 p_global=Pg, inv_temperature=invT)["stats"][1]
                lm = orc.online_dpo_loss_fwd_bwd(xm, ref, tok, mask, beta, pair_rows=pr,
                                                 p_global=Pg, inv_temperature=invT)["stats"][1]
                worst = max(worst, abs((lp - lm) / (2 * h) - rs[b, t] * G[b, t, v]))
    assert worst <= 1e-8, worst
    sm = softmax(x * np.float64(np.float32(invT)), axis=2)
    oh = np.zeros_like(sm)
    np.put_along_axis(oh, tok[..., None].astype(np.int64), 1.0, axis=2)
    live = np.zeros((B, T), bool)
    live[:4] = mask[:4] == 1
    assert np.max(np.abs(G[live] - (sm - oh)[live])) < 1e-15
    assert np.all(G[~live] == 0.0) and np.all(rs[~live] == 0.0)
    # chosen / rejected scales are opposite: coef_r = -coef_c
    assert rs[2, 0] == -rs[1, 0] and rs[0, 0] == -rs[3, 0] and rs[2, 0] > 0
    # the unscaled call's loss outputs are the scaled call's
    s_ = orc.online_dpo_loss_fwd_bwd(x, ref, tok, mask, beta, pair_rows=pr, p_global=Pg,
                                     inv_temperature=invT, want_dlogits=True)
    for k in ("seq_logp", "z", "stats"):
        assert np.array_equal(s_[k], u[k])


# ------------------------------------------------------------------------ O-9 invariants
def test_gradient_invariants(orc):
    x, tok, mask, rng = _random_batch(7, P=6, T=5, V=11)
    ref = rng.normal(-4, 1, size=12).astype(np.float32)
    out = orc.online_dpo_loss_fwd_bwd(x, ref, tok, mask, 0.1, want_dlogits=True)
    g = out["dlogits"]
    assert np.max(np.abs(g.sum(axis=2))) < 1e-15
    assert np.all(g[mask == 0] == 0.0)
    # coef_c + coef_r = 0: chosen and rejected gradients have opposite-sign tok entries
    for p in range(6):
        c, r = 2 * p, 2 * p + 1
        gc = g[c][mask[c] == 1]
        gr = g[r][mask[r] == 1]
        tc = tok[c][mask[c] == 1]
        tr = tok[r][mask[r] == 1]
        assert np.all(gc[np.arange(len(tc)), tc] <= 0) or np.all(gc[np.arange(len(tc)), tc] >= 0)
        sc = np.sign(gc[0, tc[0]])
        sr = np.sign(gr[0, tr[0]])
        assert sc == -sr


def test_unreferenced_rows_and_flags(orc):
    rng = np.random.default_rng(9)
    B, T, V = 6, 3, 8
    x = rng.normal(size=(B, T, V))
    tok = rng.integers(0, V, size=(B, T)).astype(np.int32)
    mask = np.ones((B, T), np.uint8)
    ref = np.zeros(B, np.float32)
    pr = np.array([[4, 1], [0, 5]], np.int32)
    out = orc.online_dpo_loss_fwd_bwd(x, ref, tok, mask, 0.1, pair_rows=pr, want_dlogits=True)
    assert np.all(out["dlogits"][2] == 0) and np.all(out["dlogits"][3] == 0)
    assert out["status"] == 0
    # duplicate row
    out = orc.online_dpo_loss_fwd_bwd(x, ref, tok, mask, 0.1, pair_rows=np.array([[1, 1]], np.int32))
    assert out["status"] & orc.FLAG_DUP_ROW
    out = orc.online_dpo_loss_fwd_bwd(x, ref, tok, mask, 0.1,
                                      pair_rows=np.array([[0, 1], [1, 2]], np.int32))
    assert out["status"] & orc.FLAG_DUP_ROW
    out = orc.online_dpo_loss_fwd_bwd(x, ref, tok, mask, 0.1, pair_rows=np.array([[0, 9]], np.int32))
    assert out["status"] & orc.FLAG_PAIR_RANGE
    # token out of range, NaN in masked (ignored) and unmasked (flagged) rows, empty sequence
    t2 = tok.copy()
    t2[0, 1] = V
    assert orc.seq_logprobs(x, t2, mask)["status"] & orc.FLAG_TOKEN_RANGE
    x2 = x.copy()
    x2[1, 2, 3] = np.nan
    m2 = mask.copy()
    m2[1, 2] = 0
    assert orc.seq_logprobs(x2, tok, m2)["status"] == 0
    assert orc.seq_logprobs(x2, tok, mask)["status"] & orc.FLAG_NONFINITE_LOGIT
    m3 = mask.copy()
    m3[4] = 0
    o = orc.seq_logprobs(x, tok, m3)
    assert o["status"] & orc.FLAG_EMPTY_SEQ and o["seq_logp"][4] == 0.0


# -------------------------------------------------------------------- O-10 decomposition
@pytest.mark.parametrize("W", [2, 4, 8])
def test_shard_decomposition(orc, W):
    """Pairs are independent: per-shard stats with the static P_global
    sum to the unsharded stats, and shard dlogits rows equal the unsharded rows."""
    P = 64
    x, tok, mask, rng = _random_batch(13, P=P, T=4, V=9)
    ref = rng.normal(-4, 1, size=2 * P).astype(np.float32)
    full = orc.online_dpo_loss_fwd_bwd(x, ref, tok, mask, 0.03, want_dlogits=True)
    acc = np.zeros(10)
    for r in range(W):
        p0, p1 = r * P // W, (r + 1) * P // W
        sl = slice(2 * p0, 2 * p1)
        o = orc.online_dpo_loss_fwd_bwd(np.ascontiguousarray(x[sl]), ref[sl], tok[sl], mask[sl], 0.03,
                                        p_global=P, want_dlogits=True)
        acc += o["stats"]
        assert np.array_equal(o["dlogits"], full["dlogits"][sl])
        assert np.array_equal(o["z"], full["z"][p0:p1])
    assert np.allclose(acc, full["stats"], rtol=1e-12, atol=1e-12)
    for i in (0, 2, 8, 9):
        assert acc[i] == full["stats"][i]


def test_dl_rows_subset_matches_full(orc):
    x, tok, mask, rng = _random_batch(21, P=5, T=4, V=7)
    ref = rng.normal(-4, 1, size=10).astype(np.float32)
    full = orc.online_dpo_loss_fwd_bwd(x, ref, tok, mask, 0.1, want_dlogits=True)
    rows = np.array([3, 17, 0, 39], np.int64)
    sub = orc.online_dpo_loss_fwd_bwd(x, ref, tok, mask, 0.1, dl_rows=rows)
    assert np.array_equal(sub["dlogits"], full["dlogits"].reshape(-1, 7)[rows])


def test_neg_inf_reading_r14(orc):
    """Reading R14: -inf marks an impossible token (probability 0) and is legal;
    NaN, +inf, an all -inf row, or a -inf sampled logit are flagged."""
    x = np.array([[[0.0, -np.inf, 1.0], [-np.inf, -np.inf, -np.inf]]])
    tok = np.array([[0, 1]], np.int32)
    m1 = np.array([[1, 0]], np.uint8)
    o = orc.seq_logprobs(x, tok, m1)
    assert o["status"] == 0
    assert abs(o["tok_logp"][0, 0] - (0.0 - math.log(1.0 + math.e))) < 1e-15
    assert orc.seq_logprobs(x, tok, np.array([[0, 1]], np.uint8))["status"] & orc.FLAG_NONFINITE_LOGIT
    x2 = np.array([[[0.0, -np.inf, 1.0]]])
    assert orc.seq_logprobs(x2, np.array([[1]], np.int32), np.ones((1, 1), np.uint8))["status"] \
        & orc.FLAG_NONFINITE_LOGIT
    x3 = np.array([[[0.0, np.inf, 1.0]]])
    assert orc.seq_logprobs(x3, np.array([[0]], np.int32), np.ones((1, 1), np.uint8))["status"] \
        & orc.FLAG_NONFINITE_LOGIT


# --------------------------------------------- O-10 coefficient-variant losses (App B, NEXT-3)
def _pg_batch(seed, B=6, T=3, V=5):
    rng = np.random.default_rng(seed)
    x = rng.normal(0, 1.5, size=(B, T, V))
    tok = rng.integers(0, V, size=(B, T)).astype(np.int32)
    mask = np.ones((B, T), np.uint8)
    mask[1, 2] = 0
    rew = rng.normal(0, 1, size=B).astype(np.float32)
    pr = np.array([[2, 1], [0, 3]], np.int32)    # rows 4, 5 unreferenced
    return x, tok, mask, rew, pr


def _pg_fd(orc, x, tok, mask, kind, rew, old, pr, Pg, invT, eps, g, rows_b):
    h = 1e-6
    worst = 0.0
    B, T, V = x.shape
    for b in rows_b:
        for t in range(T):
            for v in range(V):
                xp = x.copy()
                xp[b, t, v] += h
                xm = x.copy()
                xm[b, t, v] -= h
                lp = orc.pg_loss_fwd_bwd(xp, tok, mask, kind, rew, old, eps, pr, Pg, invT)["stats"][1]
                lm = orc.pg_loss_fwd_bwd(xm, tok, mask, kind, rew, old, eps, pr, Pg, invT)["stats"][1]
                worst = max(worst, abs((lp - lm) / (2 * h) - g[b, t, v]))
    return worst


@pytest.mark.parametrize("kind", ["rloo", "copg", "prox_rloo", "sft"])
def test_pg_gradient_finite_differences(orc, kind):
    """dlogits of every App B loss is the central-difference gradient of its loss value."""
    x, tok, mask, rew, pr = _pg_batch(21)
    invT, Pg, eps = 1 / 0.7, 3, 0.2
    S = orc.seq_logprobs(x, tok, mask, inv_temperature=invT)["seq_logp"]
    # old log-probs: sequence 2 inside the clip range, 1 above it, 0 and 3 below it
    # (differentiable points: |log r - log(1 +- eps)| >= 0.05)
    old = S.copy()
    old[2] -= 0.05
    old[1] -= 0.6
    old[0] += 0.6
    old[3] += 0.7
    old = old.astype(np.float32)
    out = orc.pg_loss_fwd_bwd(x, tok, mask, kind, rew, old, eps, pr, Pg, invT, want_dlogits=True)
    g = out["dlogits"]
    assert _pg_fd(orc, x, tok, mask, kind, rew, old, pr, Pg, invT, eps, g, range(4)) <= 1e-8
    assert np.all(g[4:] == 0.0) and np.all(g[1, 2] == 0.0)
    if kind == "sft":
        assert np.all(g[[1, 3]] == 0.0)     # rejected completions carry no gradient
        assert abs(out["stats"][1] + (S[2] + S[0]) / Pg) < 1e-12


def test_copg_has_the_rloo_gradient(orc):
    """CoPG and RLOO have the same gradient; their losses differ by the
    old-policy term."""
    x, tok, mask, rew, pr = _pg_batch(22)
    old = np.array([-3.0, -4.0, -5.0, -6.0, 0.0, 0.0], np.float32)
    a = orc.pg_loss_fwd_bwd(x, tok, mask, "rloo", rew, None, 0.2, pr, want_dlogits=True)
    b = orc.pg_loss_fwd_bwd(x, tok, mask, "copg", rew, old, 0.2, pr, want_dlogits=True)
    assert np.array_equal(a["dlogits"], b["dlogits"])
    r64, o64 = rew.astype(np.float64), old.astype(np.float64)
    A = [r64[2] - r64[1], r64[0] - r64[3]]
    shift = 0.5 * sum(A[i] * (o64[pr[i, 0]] - o64[pr[i, 1]]) for i in range(2)) / 2
    assert abs((b["stats"][1] - a["stats"][1]) - shift) < 1e-12


def test_prox_rloo_special_cases(orc):
    """r = 1 (pi_old = pi_theta): the RLOO gradient and a zero loss (A2 = -A1); a ratio
    outside the clip range on the improving side: zero gradient, loss at the clipped value."""
    x, tok, mask, rew, pr = _pg_batch(23)
    S = orc.seq_logprobs(x, tok, mask)["seq_logp"]
    old = S.astype(np.float32)
    S32 = old.astype(np.float64)
    r = orc.pg_loss_fwd_bwd(x, tok, mask, "rloo", rew, None, 0.2, pr, want_dlogits=True)
    p = orc.pg_loss_fwd_bwd(x, tok, mask, "prox_rloo", rew, old, 0.2, pr, want_dlogits=True)
    ratio = np.exp(S - S32)           # 1 up to the f32 rounding of old_logp
    assert np.max(np.abs(ratio - 1)) < 1e-6
    assert np.max(np.abs(p["dlogits"] - r["dlogits"])) < 1e-6 * np.max(np.abs(r["dlogits"]))
    assert abs(p["stats"][1]) < 1e-6 and p["stats"][2] == 4
    # sequence 2 (chosen of pair 0) with A > 0 and r = e^0.5 > 1.2: clipped, no gradient
    A0 = float(rew[2]) - float(rew[1])
    old2 = old.copy()
    old2[2] = np.float32(S[2] - 0.5) if A0 > 0 else np.float32(S[2] + 0.5)
    q = orc.pg_loss_fwd_bwd(x, tok, mask, "prox_rloo", rew, old2, 0.2, pr, want_dlogits=True)
    assert np.all(q["dlogits"][2] == 0.0) and q["stats"][2] == 3
    assert np.array_equal(q["dlogits"][[0, 1, 3]], p["dlogits"][[0, 1, 3]]) or \
        np.max(np.abs(q["dlogits"][[0, 1, 3]] - p["dlogits"][[0, 1, 3]])) < 1e-15


def test_rloo_uniform_rows_closed_form(orc):
    """Uniform rows: S_b = -n_b log V, so the RLOO loss is -1/2 sum_p A_p (S_1 - S_2) / P."""
    B, T, V = 4, 3, 7
    x = np.zeros((B, T, V))
    tok = np.zeros((B, T), np.int32)
    mask = np.array([[1, 1, 1], [1, 0, 0], [1, 1, 0], [1, 1, 1]], np.uint8)
    rew = np.array([1.0, -0.5, 0.25, 2.0], np.float32)
    out = orc.pg_loss_fwd_bwd(x, tok, mask, "rloo", rew, None, 0.2)
    S = -mask.sum(1).astype(np.float64) * np.log(V)
    A = [1.5, -1.75]
    want = (-0.5 * (A[0] * (S[0] - S[1]) + A[1] * (S[2] - S[3]))) / 2
    assert abs(out["stats"][1] - want) < 1e-12


@pytest.mark.parametrize("kind", ["rloo", "sft"])
def test_pg_shard_decomposition(orc, kind):
    """App B losses shard like DPO: with a static P_global, per-shard loss stats sum to the
    unsharded ones and shard gradients equal the unsharded rows (weak-scaling invariance)."""
    rng = np.random.default_rng(31)
    P, T, V, W = 6, 3, 9, 3
    x = rng.normal(0, 1.2, size=(2 * P, T, V))
    tok = rng.integers(0, V, size=(2 * P, T)).astype(np.int32)
    mask = np.ones((2 * P, T), np.uint8)
    rew = rng.normal(0, 1, size=2 * P).astype(np.float32)
    full = orc.pg_loss_fwd_bwd(x, tok, mask, kind, rew, None, 0.2, None, P, 1.0, want_dlogits=True)
    acc = np.zeros(10)
    for r in range(W):
        sl = slice(2 * P * r // W, 2 * P * (r + 1) // W)
        o = orc.pg_loss_fwd_bwd(x[sl], tok[sl], mask[sl], kind, rew[sl], None, 0.2, None, P, 1.0,
                                want_dlogits=True)
        acc += o["stats"]
        assert np.array_equal(o["dlogits"], full["dlogits"][sl])
    assert np.allclose(acc, full["stats"], rtol=1e-12, atol=1e-12)
