"""Shared builders for the GPU parity tests: seeded synthetic inputs drawn once from
``synth`` and handed to BOTH the CUDA path (device tensors) and the CPU oracle (host
arrays).  Tolerances follow SURVEY.md §8(c) / DESIGN.md section 7."""
from __future__ import annotations

import os

import numpy as np
import torch

import oracle
import synth

NCPU = os.cpu_count() or 1

TOL_SEQ = {"f32": 1e-5, "bf16": 2e-3}            # north_star: 1e-5 fp32, 2e-3 bf16 (relative)
DL_RTOL = {"f32": 1e-5, "bf16": 2.0 ** -7}   # bf16: faithful rounding, one ulp (DESIGN R17)
DL_ATOL = {"f32": 1e-7, "bf16": 2.0 ** -20}      # times |coef_b|
TORCH_DT = {"f32": torch.float32, "bf16": torch.bfloat16}


def alloc_rows(B, T, V, dtype, device="cuda"):
    """[B, T, V] view whose row stride is padded to a multiple of 16 bytes (the C ABI's
    128-bit alignment contract; V itself may be ragged)."""
    es = 4 if dtype == "f32" else 2
    vp = -(-V * es // 16) * 16 // es
    return torch.empty((B, T, vp), dtype=TORCH_DT[dtype], device=device)[:, :, :V]


class Batch:
    """One synthetic Online-DPO batch: P pairs, rows (2p, 2p+1) unless perm is given."""

    def __init__(self, P, T, V, dtype="bf16", seed=0, mask_kind="dense", lbar=None, peak=14.0,
                 p0=0, extra_seqs=0, permute=False, device="cuda", host=True, invT=1.0):
        self.P, self.T, self.V, self.dtype, self.seed = P, T, V, dtype, seed
        self.B = 2 * P + extra_seqs
        self.invT = invT
        B = self.B
        seqs = np.arange(B) + 2 * p0
        rows = (seqs[:, None] * T + np.arange(T)[None, :]).reshape(-1)
        self.rows_global = rows
        self.tokens = synth.tokens_rows(seed, rows, V).reshape(B, T)
        self.mask = synth.mask_for(seed, seqs, T, mask_kind, lbar)
        self.peak = peak
        if permute or extra_seqs:
            perm = synth.permutation(seed, B)
            self.pair_rows = perm[: 2 * P].reshape(P, 2).astype(np.int32)
        else:
            self.pair_rows = None
        dev = torch.device(device)
        self.d_tokens = torch.from_numpy(self.tokens).to(dev)
        self.d_mask = torch.from_numpy(self.mask).to(dev)
        self.d_pair_rows = None if self.pair_rows is None else torch.from_numpy(self.pair_rows).to(dev)
        self.d_logits = alloc_rows(B, T, V, dtype, dev)
        synth.fill_logits_device(self.d_logits, seed, row0=int(rows[0]), tokens=self.d_tokens,
                                 peak=peak)
        self.h_logits = None
        if host:
            self.h_logits = self.host_rows(np.arange(B))

    def new_out(self):
        """An output buffer with the same (16-byte aligned, padded) row layout."""
        return alloc_rows(self.B, self.T, self.V, self.dtype, self.d_logits.device)

    def host_rows(self, seqs):
        """Host logits [len(seqs), T, V] in the oracle's input encoding (f32 or bf16 bits).
        Rows with mask 0 are never read by either side and are left at zero."""
        seqs = np.asarray(seqs)
        rows = (seqs[:, None] * self.T + np.arange(self.T)[None, :]).reshape(-1)
        live = self.mask.reshape(-1)[rows] == 1
        x = np.zeros((rows.size, self.V))
        x[live] = synth.logits_rows(self.seed, self.rows_global[rows[live]], self.V,
                                    tokens=self.tokens.reshape(-1)[rows[live]], peak=self.peak)
        x = x.reshape(len(seqs), self.T, self.V)
        if self.dtype == "f32":
            return x.astype(np.float32)
        return oracle.to_bf16_bits(x.astype(np.float32))


def check_seq(gpu, orc, dtype, what="seq_logp"):
    gpu = np.asarray(gpu, dtype=np.float64)
    tol = TOL_SEQ[dtype]
    err = np.abs(gpu - orc)
    bound = tol * np.maximum(np.abs(orc), 1.0)
    assert np.all(err <= bound), f"{what}: max rel err {np.max(err / np.maximum(np.abs(orc), 1.0)):.3e}"
    return float(np.max(err / np.maximum(np.abs(orc), 1.0))) if err.size else 0.0


def check_dlogits(g_gpu, g_orc, coef_abs, dtype):
    """|g_gpu - g_orc| <= rtol |g_orc| + atol |coef_b| per element (coef_abs broadcast per row)."""
    g_gpu = np.asarray(g_gpu, dtype=np.float64)
    err = np.abs(g_gpu - g_orc)
    bound = DL_RTOL[dtype] * np.abs(g_orc) + DL_ATOL[dtype] * coef_abs
    bad = err > bound
    assert not np.any(bad), (
        f"dlogits: {np.count_nonzero(bad)} elements out of tolerance; "
        f"worst excess {np.max(err - bound):.3e}")


def to_f64(t: torch.Tensor) -> np.ndarray:
    return t.detach().float().cpu().double().numpy()


def coef_from_oracle(o, P, Pg, beta, invT, pair_rows, B):
    """|coef_b| per sequence from the oracle's z (for the dlogits absolute tolerance)."""
    coef = np.zeros(B)
    beta = float(np.float32(beta))
    for p in range(P):
        c, r = (2 * p, 2 * p + 1) if pair_rows is None else pair_rows[p]
        sig = 1.0 / (1.0 + np.exp(o["z"][p]))
        coef[c] = coef[r] = beta * sig * float(np.float32(invT)) / Pg
    return coef


def pair_members(P, pair_rows):
    if pair_rows is None:
        return np.arange(P) * 2, np.arange(P) * 2 + 1
    pr = np.asarray(pair_rows).reshape(-1, 2)
    return pr[:, 0].astype(np.int64), pr[:, 1].astype(np.int64)


def check_stats(st_gpu, o, dtype, beta, ref, pair_rows=None, Pg=None, exact_ncorrect=None,
                tol=None):
    """All ten loss statistics (ODPO_ST_*) against the oracle.

    Counts (npairs, token counts) are exact; ncorrect is exact wherever no oracle |z| lies
    inside the per-pair error band (else within the number of pairs in the band).  Every
    float statistic is a sum of per-pair terms; its bound is the sum of the per-pair bounds
    propagated from the north_star sequence tolerance (|dS_b| <= tol max(|S_b|, 1 nat))
    plus the fp32 roundings of S, S - ref and z:
      S sums:            sum tol max(|S|, 1) + 2^-24 |S|
      beta (S - ref):    beta x (the above + 2^-24 (|S| + |ref|))
      z:                 beta (e_c + e_r) + 2^-23 |z|
      loss (/P_global):  sum e_z / P_global  (|d softplus(-z) / dz| <= 1)."""
    st = np.asarray(st_gpu, dtype=np.float64)[:10]
    os_ = np.asarray(o["stats"], dtype=np.float64)
    S = np.asarray(o["seq_logp"], dtype=np.float64)
    z = np.asarray(o["z"], dtype=np.float64)
    P = z.size
    Pg = P if Pg is None else Pg
    c, r = pair_members(P, pair_rows)
    tol = TOL_SEQ[dtype] if tol is None else tol
    ref = np.asarray(ref, dtype=np.float64)
    b = float(np.float32(beta))
    eS_c = tol * np.maximum(np.abs(S[c]), 1.0) + 2.0 ** -24 * np.abs(S[c])
    eS_r = tol * np.maximum(np.abs(S[r]), 1.0) + 2.0 ** -24 * np.abs(S[r])
    ed_c = eS_c + 2.0 ** -24 * (np.abs(S[c]) + np.abs(ref[c]))
    ed_r = eS_r + 2.0 ** -24 * (np.abs(S[r]) + np.abs(ref[r]))
    ez = b * (ed_c + ed_r) + 2.0 ** -23 * np.abs(z)
    bounds = {1: ez.sum() / Pg, 3: ez.sum(), 4: b * ed_c.sum(), 5: b * ed_r.sum(),
              6: eS_c.sum(), 7: eS_r.sum()}
    for i in (0, 8, 9):
        assert st[i] == os_[i], (i, st[i], os_[i])
    band = np.count_nonzero(np.abs(z) <= ez)
    if exact_ncorrect is None:
        exact_ncorrect = band == 0
    if exact_ncorrect:
        assert st[2] == os_[2], ("ncorrect", st[2], os_[2])
    else:
        assert abs(st[2] - os_[2]) <= band, ("ncorrect", st[2], os_[2], band)
    for i, bd in bounds.items():
        assert abs(st[i] - os_[i]) <= bd + 1e-12, (i, st[i], os_[i], bd)


def controlled_ref(S_orc, P, pair_rows, seed):
    """Controlled-ref mode: ref = fl32(S - delta) with delta_r = 0 and
    delta_c = +-(1 + h % 128)/16, so z ~ beta delta_c is never inside the fp error band.
    S_orc is the ORACLE's sequence log-prob (an input to both sides)."""
    c, _ = pair_members(P, pair_rows)
    h = synth.uniform_u32(seed, synth.S_DELTA, np.arange(P))
    delta = np.zeros(S_orc.size)
    delta[c] = np.where(h & 1, 1.0, -1.0) * (1 + (h >> 1) % 128) / 16.0
    return (S_orc - delta).astype(np.float32)


def to_device_logits(h, dtype):
    """Host logits in the oracle's encoding (float32 or bf16 bits) -> a padded device view."""
    B, T, V = h.shape
    d = alloc_rows(B, T, V, dtype)
    if dtype == "f32":
        d.copy_(torch.from_numpy(np.ascontiguousarray(h)))
    else:
        d.copy_(torch.from_numpy(np.ascontiguousarray(h).view(np.int16)).view(torch.bfloat16))
    return d
