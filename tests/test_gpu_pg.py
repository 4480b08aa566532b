"""GPU-vs-oracle parity of the App B coefficient-variant losses (odpo_pg_loss_fwd_bwd;
SURVEY.md §8 NEXT-3): RLOO, CoPG, Proximal RLOO and Best-of-2 SFT on the same kernels."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_helpers import DL_RTOL, NCPU, TOL_SEQ, Batch, check_dlogits, check_seq, to_f64

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

KINDS = ["rloo", "copg", "prox_rloo", "sft"]


@pytest.fixture(scope="module")
def odpo():
    import paper_2410_18252_b200 as m
    m._L()
    return m


def pg_inputs(b: Batch, seed):
    """Per-sequence rewards and old log-probs.  old = S_oracle + offset with offsets 0.05 (ratio
    inside the clip range) or +-0.6 (outside), so no clip decision sits near a boundary."""
    rew = (synth.rewards_for(seed, b.B, 1).reshape(-1)).astype(np.float32)
    S = oracle.seq_logprobs(b.h_logits, b.tokens, b.mask, inv_temperature=b.invT,
                            n_threads=NCPU)["seq_logp"]
    off = np.array([-0.05, 0.6, -0.6, 0.05])[np.arange(b.B) % 4]
    return rew, (S + off).astype(np.float32)



def coef_bound(rew, old, S, invT, Pg, B, pair_rows):
    """Upper bound on |coef_b| for every kind (the absolute part of the dlogits tolerance)."""
    pr = np.arange(B).reshape(-1, 2) if pair_rows is None else pair_rows
    bound = np.zeros(B)
    for c, r in pr:
        A = abs(float(rew[c]) - float(rew[r]))
        for b in (c, r):
            ratio = np.exp(S[b] - old[b]) if old is not None else 1.0
            bound[b] = (A * max(1.0, ratio) + 2.0) * invT / Pg
    return bound


CASES = [
    (3, 5, 4133, "bf16", "prefix", 2, 1.0),
    (3, 5, 4133, "f32", "prefix", 1, 1 / 0.7),
    (4, 9, 32000, "bf16", "dense", 0, 1.0),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"P{c[0]}T{c[1]}V{c[2]}{c[3]}x{c[5]}")
@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("sched", ["auto", "two_pass"])
def test_pg_parity_small(odpo, case, kind, sched):
    if sched == "two_pass" and kind != "prox_rloo":
        pytest.skip("the schedule option applies to Proximal RLOO only")
    P, T, V, dt, mk, extra, invT = case
    b = Batch(P, T, V, dt, seed=4, mask_kind=mk, lbar=max(1, T // 2), extra_seqs=extra, invT=invT)
    rew, old = pg_inputs(b, 4)
    Pg, eps = P + 2, 0.2
    out = odpo.pg_loss_fwd_bwd(b.d_logits, b.d_tokens, b.d_mask, kind, torch.from_numpy(rew).cuda(),
                               torch.from_numpy(old).cuda(), eps, pair_rows=b.d_pair_rows,
                               p_global=Pg, inv_temperature=invT, dlogits=b.new_out(),
                               schedule=sched)
    torch.cuda.synchronize()
    o = oracle.pg_loss_fwd_bwd(b.h_logits, b.tokens, b.mask, kind, rew, old, eps, b.pair_rows, Pg,
                               invT, want_dlogits=True, n_threads=NCPU)
    live = np.arange(b.B) if b.pair_rows is None else b.pair_rows.reshape(-1)
    check_seq(out.seq_logp.cpu().numpy()[live], o["seq_logp"][live], dt)
    st = out.stats.cpu().numpy()
    assert st[0] == o["stats"][0] and st[2] == o["stats"][2]
    assert st[8] == o["stats"][8] and st[9] == o["stats"][9]
    assert abs(st[4] - o["stats"][4]) <= 1e-6 * max(1.0, abs(o["stats"][4]))
    # loss: absolute floor scaled by the advantages (a loss can cancel to ~0)
    lt = TOL_SEQ[dt] * max(abs(o["stats"][1]), np.abs(rew).max() * np.abs(o["seq_logp"]).max() / Pg)
    assert abs(st[1] - o["stats"][1]) <= lt, (st[1], o["stats"][1])
    cb = coef_bound(rew, old, o["seq_logp"], invT, Pg, b.B, b.pair_rows)
    check_dlogits(to_f64(out.dlogits), o["dlogits"], cb[:, None, None], dt)
    assert int(out.status.item()) == 0


def test_pg_single_pass_launches_and_zero_rows(odpo):
    """RLOO / CoPG / SFT know their coefficients before the forward: prep + coef + one engine
    launch; SFT's rejected completions and unreferenced sequences get exact zeros."""
    b = Batch(4, 7, 5001, "bf16", seed=9, extra_seqs=2, host=False)
    rew = torch.linspace(-1, 1, b.B, device="cuda")
    out = odpo.pg_loss_fwd_bwd(b.d_logits, b.d_tokens, b.d_mask, "sft", rew,
                               pair_rows=b.d_pair_rows, dlogits=b.new_out())
    torch.cuda.synchronize()
    assert out.launches == 3
    rej = b.d_pair_rows[:, 1].long()
    assert torch.count_nonzero(out.dlogits[rej]).item() == 0
    unref = np.setdiff1d(np.arange(b.B), b.pair_rows.reshape(-1))
    assert torch.count_nonzero(out.dlogits[torch.from_numpy(unref).cuda()]).item() == 0
    prox = odpo.pg_loss_fwd_bwd(b.d_logits, b.d_tokens, b.d_mask, "prox_rloo", rew,
                                torch.zeros(b.B, device="cuda"), 0.2, pair_rows=b.d_pair_rows,
                                dlogits=b.new_out())
    torch.cuda.synchronize()
    assert prox.launches == 2


def test_rloo_full_size_pythia_sampled(odpo):
    """Pythia TLDR shape at full size, RLOO (single pass): sampled pairs against the oracle."""
    from synth.configs import CONFIGS
    w = CONFIGS["pythia"]
    b = Batch(w.P, w.T, w.V, w.dtype, seed=0, host=False)
    rew = synth.rewards_for(0, w.P, 2).reshape(-1).astype(np.float32)
    out = odpo.pg_loss_fwd_bwd(b.d_logits, b.d_tokens, b.d_mask, "rloo",
                               torch.from_numpy(rew).cuda())
    torch.cuda.synchronize()
    pairs = synth.permutation(2, w.P)[:2]
    seqs = np.stack([2 * pairs, 2 * pairs + 1], 1).reshape(-1)
    h_x = b.host_rows(seqs)
    rows = (np.arange(len(seqs))[:, None] * w.T + np.arange(w.T)[None, :])[:, :3].reshape(-1)
    o = oracle.pg_loss_fwd_bwd(h_x, b.tokens[seqs], b.mask[seqs], "rloo", rew[seqs], None, 0.2,
                               None, w.P, 1.0, dl_rows=rows, n_threads=NCPU)
    check_seq(out.seq_logp.cpu().numpy()[seqs], o["seq_logp"], w.dtype)
    gi = torch.from_numpy(seqs).cuda()
    g = to_f64(out.dlogits[gi][:, :3].reshape(-1, w.V))
    cb = np.repeat(coef_bound(rew[seqs], None, o["seq_logp"], 1.0, w.P, len(seqs), None), 3)
    check_dlogits(g, o["dlogits"], cb[:, None], w.dtype)
    assert out.stats[0].item() == w.P and int(out.status.item()) == 0
    del b, out
    torch.cuda.empty_cache()
