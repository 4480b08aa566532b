"""Edge cases of the hot path against the oracle (the task's "empty and ragged inputs, maximum
sizes, the degenerate cases the method has"): vocabularies of 1..15 entries (V = 1: every
log-prob is exactly 0 and every dlogit 0; V below one 16-byte vector: only the scalar tail),
single-token responses, a single pair, fully masked sequences (EMPTY_SEQ, S = 0), extreme
inverse temperatures, ties and wide groups in pair selection (K up to 16), and sequences
with only one live token at the row's last vocabulary entry."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_helpers import (NCPU, check_dlogits, check_seq, check_stats, coef_from_oracle,
                         controlled_ref, to_device_logits, to_f64)

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def odpo():
    import paper_2410_18252_b200 as m
    m._L()
    return m


def _case(P, T, V, dtype, seed, kind="grid"):
    B = 2 * P
    tok = synth.tokens_rows(seed, np.arange(B * T), V).reshape(B, T).astype(np.int32)
    if kind == "grid":
        x = synth.logits_rows(seed, np.arange(B * T), V, tokens=tok.reshape(-1)).reshape(B, T, V)
    else:
        x = np.random.default_rng(seed).normal(0.0, 3.0, size=(B, T, V))
    h = x.astype(np.float32) if dtype == "f32" else oracle.to_bf16_bits(x.astype(np.float32))
    return B, tok, h


def _run(odpo, sched, d, ref, tok, mask, beta, invT=1.0, Pg=None):
    args = (d, torch.from_numpy(ref).cuda(), torch.from_numpy(tok).cuda(),
            torch.from_numpy(mask).cuda(), beta)
    kw = dict(inv_temperature=invT, p_global=Pg)
    if sched == "unscaled":
        out = odpo.online_dpo_loss_fwd_bwd_unscaled(*args, **kw)
    else:
        out = odpo.online_dpo_loss_fwd_bwd(*args, schedule=sched, **kw)
    torch.cuda.synchronize()
    return out


SMALL = [(1, 1, 1), (1, 1, 2), (2, 1, 7), (1, 3, 9), (3, 2, 15), (1, 4, 17)]


@pytest.mark.parametrize("shape", SMALL, ids=lambda s: f"P{s[0]}T{s[1]}V{s[2]}")
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("sched", ["fused", "two_pass", "unscaled"])
def test_tiny_vocabularies_and_lengths(odpo, shape, dtype, sched):
    P, T, V = shape
    B, tok, h = _case(P, T, V, dtype, seed=41, kind="normal")
    mask = np.ones((B, T), np.uint8)
    S = oracle.seq_logprobs(h, tok, mask)["seq_logp"]
    ref = controlled_ref(S, P, None, 41)
    beta = 0.1
    out = _run(odpo, sched, to_device_logits(h, dtype), ref, tok, mask, beta, Pg=P + 1)
    o = oracle.online_dpo_loss_fwd_bwd(h, ref, tok, mask, beta, p_global=P + 1, want_dlogits=True,
                                       unscaled=(sched == "unscaled"))
    assert int(out.status.item()) == 0
    check_seq(out.seq_logp.cpu().numpy(), o["seq_logp"], dtype)
    check_stats(out.stats.cpu().numpy(), o, dtype, beta, ref, None, Pg=P + 1, exact_ncorrect=True)
    if V == 1:
        # a one-entry vocabulary: log p = 0 exactly, the gradient vanishes
        assert np.all(out.seq_logp.cpu().numpy() == 0.0)
        assert torch.count_nonzero(out.dlogits).item() == 0
    if sched == "unscaled":
        check_dlogits(to_f64(out.dlogits), o["dlogits"], np.ones((B, 1, 1)), dtype)
    else:
        coef = coef_from_oracle(o, P, P + 1, beta, 1.0, None, B)
        check_dlogits(to_f64(out.dlogits), o["dlogits"], coef[:, None, None], dtype)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_fully_masked_sequence(odpo, dtype):
    """A completion with no response token: EMPTY_SEQ is flagged, its log-prob is 0 (SPEC
    "empty completion -> error", DESIGN R4), its dlogits rows are zeros, the pair's other
    sequence and every other pair are unaffected."""
    P, T, V = 3, 6, 4133
    B, tok, h = _case(P, T, V, dtype, seed=42)
    mask = synth.mask_for(42, np.arange(B), T, "prefix", 3)
    mask[3] = 0
    ref = np.full(B, -2.0, np.float32)
    beta = 0.1
    out = _run(odpo, "fused", to_device_logits(h, dtype), ref, tok, mask, beta)
    o = oracle.online_dpo_loss_fwd_bwd(h, ref, tok, mask, beta, want_dlogits=True)
    assert int(out.status.item()) & odpo.FLAGS["EMPTY_SEQ"]
    assert o["status"] & oracle.FLAG_EMPTY_SEQ
    assert out.seq_logp[3].item() == 0.0
    assert torch.count_nonzero(out.dlogits[3]).item() == 0
    check_seq(out.seq_logp.cpu().numpy(), o["seq_logp"], dtype)
    coef = coef_from_oracle(o, P, P, beta, 1.0, None, B)
    check_dlogits(to_f64(out.dlogits), o["dlogits"], coef[:, None, None], dtype)
    st = out.stats.cpu().numpy()
    assert st[0] == o["stats"][0] and st[8] == o["stats"][8] and st[9] == o["stats"][9]


@pytest.mark.parametrize("invT", [0.25, 1 / 0.7, 4.0])
def test_inverse_temperature_extremes(odpo, invT):
    P, T, V = 2, 5, 12345
    B, tok, h = _case(P, T, V, "f32", seed=43)
    mask = np.ones((B, T), np.uint8)
    S = oracle.seq_logprobs(h, tok, mask, inv_temperature=invT)["seq_logp"]
    ref = controlled_ref(S, P, None, 43)
    beta = 0.05
    out = _run(odpo, "fused", to_device_logits(h, "f32"), ref, tok, mask, beta, invT=invT)
    o = oracle.online_dpo_loss_fwd_bwd(h, ref, tok, mask, beta, inv_temperature=invT,
                                       want_dlogits=True)
    check_seq(out.seq_logp.cpu().numpy(), o["seq_logp"], "f32")
    check_stats(out.stats.cpu().numpy(), o, "f32", beta, ref, None, exact_ncorrect=True)
    coef = coef_from_oracle(o, P, P, beta, invT, None, B)
    check_dlogits(to_f64(out.dlogits), o["dlogits"], coef[:, None, None], "f32")


@pytest.mark.parametrize("K", [5, 8, 16])
def test_pair_select_wide_groups(odpo, K):
    """Best/worst of K for wide groups, with heavy ties (verifier rewards) and
    EOS penalties: bit-exact selection, margins and statistics at the strong config's 2048
    prompts."""
    for kind, pen in (("rm", -10.0), ("verifier", -1.0)):
        rewards = synth.rewards_for(44, 2048, K, kind=kind)
        eos = synth.has_eos_for(44, 2048, K)
        g = odpo.pair_select(torch.from_numpy(rewards).cuda(), torch.from_numpy(eos).cuda(), pen)
        o = oracle.pair_select(rewards, eos, pen)
        assert np.array_equal(g.pair_rows.cpu().numpy(), o["pair_rows"])
        assert np.array_equal(g.reward_margin.cpu().numpy().view(np.uint32),
                              o["margin"].view(np.uint32))
        s = g.sel_stats.cpu().numpy()
        assert s[1] == o["sel_stats"][1] and s[2] == o["sel_stats"][2]
        assert int(g.status.item()) == o["status"]


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_token_at_the_last_vocabulary_entry(odpo, dtype):
    """Every sampled token is V - 1 (the row's scalar tail when V is not a multiple of the
    vector width): the gather, the tail of the online log-sum-exp and the onehot entry of the
    backward all hit the ragged end of the row."""
    P, T, V = 2, 4, 4133
    B = 2 * P
    tok = np.full((B, T), V - 1, np.int32)
    x = synth.logits_rows(45, np.arange(B * T), V, tokens=tok.reshape(-1)).reshape(B, T, V)
    h = x.astype(np.float32) if dtype == "f32" else oracle.to_bf16_bits(x.astype(np.float32))
    mask = np.ones((B, T), np.uint8)
    S = oracle.seq_logprobs(h, tok, mask)["seq_logp"]
    ref = controlled_ref(S, P, None, 45)
    out = _run(odpo, "fused", to_device_logits(h, dtype), ref, tok, mask, 0.1)
    o = oracle.online_dpo_loss_fwd_bwd(h, ref, tok, mask, 0.1, want_dlogits=True)
    check_seq(out.seq_logp.cpu().numpy(), o["seq_logp"], dtype)
    coef = coef_from_oracle(o, P, P, 0.1, 1.0, None, B)
    check_dlogits(to_f64(out.dlogits), o["dlogits"], coef[:, None, None], dtype)
