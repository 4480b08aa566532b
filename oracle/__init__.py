"""ctypes shim over the CPU oracle ``oracle/liboracle.so`` (see oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs.  The product package
``paper_2410_18252_b200`` never imports this module.

Arrays are numpy.  Logits may be float32 (F32), float64 (F64, oracle-only, used
for finite differences) or uint16 holding bf16 bit patterns (BF16).  Strided
logits ([B, T', V'] views whose last dimension is contiguous) are passed with
their element strides.  Every float result comes back as float64 so comparisons
happen before any rounding.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

F32, BF16, F64 = 0, 1, 2
FLAG_TOKEN_RANGE, FLAG_NONFINITE_LOGIT, FLAG_EMPTY_SEQ = 1, 2, 4
FLAG_NONFINITE_REWARD, FLAG_DUP_ROW, FLAG_DEGENERATE_PAIR, FLAG_PAIR_RANGE = 8, 16, 32, 64
ST_NAMES = ["npairs", "loss", "ncorrect", "z_sum", "rchosen_sum", "rrej_sum",
            "schosen_sum", "srej_sum", "ntok_chosen", "ntok_rej"]
SEL_NAMES = ["margin_sum", "ndegen", "ntrunc"]

_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
                               "-fPIC", "-shared", "-o", LIB_PATH, src, "-lm", "-lpthread"])
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        i64, i32, f32 = C.c_int64, C.c_int32, C.c_float
        L.orc_pair_select.argtypes = [P, P, f32, i64, i32, P, P, P, P, P, P]
        L.orc_seq_logprobs.argtypes = [P, C.c_int, i64, i64, i64, i64, i64, P, P, f32, P, P, P, P,
                                       C.c_int]
        L.orc_online_dpo_loss_fwd_bwd.argtypes = [P, C.c_int, i64, i64, i64, i64, i64, P, P, P, P,
                                                  i64, i64, f32, f32, P, P, i64, P, P, P, P, C.c_int]
        L.orc_online_dpo_loss_fwd_bwd_unscaled.argtypes = [
            P, C.c_int, i64, i64, i64, i64, i64, P, P, P, P, i64, i64, f32, f32, P, P, i64, P, P, P,
            P, P, C.c_int]
        L.orc_pg_loss_fwd_bwd.argtypes = [P, C.c_int, i64, i64, i64, i64, i64, P, P, P, i64, i64,
                                          C.c_int, P, P, f32, f32, P, P, i64, P, P, P, C.c_int]
        L.orc_seq_ppl.argtypes = [P, C.c_int, i64, i64, i64, i64, i64, P, P, f32, P, P, P, P,
                                  C.c_int]
        for f in (L.orc_pair_select, L.orc_seq_logprobs, L.orc_online_dpo_loss_fwd_bwd,
                  L.orc_online_dpo_loss_fwd_bwd_unscaled, L.orc_pg_loss_fwd_bwd, L.orc_seq_ppl):
            f.restype = C.c_int
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _logits_args(logits):
    a = np.asarray(logits)
    if a.ndim != 3:
        raise ValueError("logits must be [B, T, V]")
    if a.dtype == np.float32:
        dt = F32
    elif a.dtype == np.float64:
        dt = F64
    elif a.dtype == np.uint16:
        dt = BF16
    else:
        raise TypeError(f"unsupported logits dtype {a.dtype}")
    isz = a.itemsize
    sb, st, sv = (s // isz for s in a.strides)
    if sv != 1 or a.strides[0] % isz or a.strides[1] % isz:
        raise ValueError("logits last dimension must be contiguous")
    return a, dt, sb, st


def pair_select(rewards, has_eos=None, eos_penalty=-1.0):
    r = np.ascontiguousarray(rewards, dtype=np.float32)
    P, K = r.shape
    e = None if has_eos is None else np.ascontiguousarray(has_eos, dtype=np.uint8)
    chosen = np.zeros(P, np.int32)
    rejected = np.zeros(P, np.int32)
    pair_rows = np.zeros((P, 2), np.int32)
    margin = np.zeros(P, np.float32)
    sel = np.zeros(3, np.float64)
    status = np.zeros(1, np.uint32)
    rc = lib().orc_pair_select(_ptr(r), _ptr(e), float(eos_penalty), P, K, _ptr(chosen),
                               _ptr(rejected), _ptr(pair_rows), _ptr(margin), _ptr(sel),
                               _ptr(status))
    if rc:
        raise ValueError("orc_pair_select: invalid argument")
    return dict(chosen=chosen, rejected=rejected, pair_rows=pair_rows, margin=margin,
                sel_stats=sel, status=int(status[0]))


def seq_logprobs(logits, tokens, mask, inv_temperature=1.0, n_threads=1):
    a, dt, sb, st = _logits_args(logits)
    B, T, V = a.shape
    tok = np.ascontiguousarray(tokens, dtype=np.int32).reshape(B, T)
    msk = np.ascontiguousarray(mask, dtype=np.uint8).reshape(B, T)
    S = np.zeros(B, np.float64)
    tlp = np.zeros((B, T), np.float64)
    lse = np.zeros((B, T), np.float64)
    status = np.zeros(1, np.uint32)
    rc = lib().orc_seq_logprobs(_ptr(a), dt, B, T, V, sb, st, _ptr(tok), _ptr(msk),
                                float(np.float32(inv_temperature)), _ptr(S), _ptr(tlp), _ptr(lse),
                                _ptr(status), int(n_threads))
    if rc:
        raise ValueError("orc_seq_logprobs: invalid argument")
    return dict(seq_logp=S, tok_logp=tlp, row_lse=lse, status=int(status[0]))


def seq_ppl(logits, tokens, mask, inv_temperature=1.0, n_threads=1):
    """KL proxy: per-completion perplexity exp(-S_b / n_b) of the model
    whose logits are given.  Returns dict(seq_logp[B], ppl[B], ppl_stats[4] = (#nonempty,
    sum ppl, sum S, sum n), status)."""
    a, dt, sb, st = _logits_args(logits)
    B, T, V = a.shape
    tok = np.ascontiguousarray(tokens, dtype=np.int32).reshape(B, T)
    msk = np.ascontiguousarray(mask, dtype=np.uint8).reshape(B, T)
    S = np.zeros(B, np.float64)
    ppl = np.zeros(B, np.float64)
    ps = np.zeros(4, np.float64)
    status = np.zeros(1, np.uint32)
    rc = lib().orc_seq_ppl(_ptr(a), dt, B, T, V, sb, st, _ptr(tok), _ptr(msk),
                           float(np.float32(inv_temperature)), _ptr(S), _ptr(ppl), _ptr(ps),
                           _ptr(status), int(n_threads))
    if rc:
        raise ValueError("orc_seq_ppl: invalid argument")
    return dict(seq_logp=S, ppl=ppl, ppl_stats=ps, status=int(status[0]))


def online_dpo_loss_fwd_bwd(logits, ref_logp, tokens, mask, beta, pair_rows=None, p_global=None,
                            inv_temperature=1.0, want_dlogits=False, dl_rows=None, n_threads=1,
                            unscaled=False):
    """Returns dict(seq_logp[B], z[P], stats[10], status, dlogits[n, V] or None).

    unscaled=True: 'dlogits' holds G = mask (softmax - onehot) (no coef_b) and 'row_scale'[B, T]
    holds coef_b * mask, so the gradient is row_scale[..., None] * G."""
    a, dt, sb, st = _logits_args(logits)
    B, T, V = a.shape
    tok = np.ascontiguousarray(tokens, dtype=np.int32).reshape(B, T)
    msk = np.ascontiguousarray(mask, dtype=np.uint8).reshape(B, T)
    ref = np.ascontiguousarray(ref_logp, dtype=np.float32).reshape(B)
    pr = None if pair_rows is None else np.ascontiguousarray(pair_rows, dtype=np.int32).reshape(-1, 2)
    P = B // 2 if pr is None else pr.shape[0]
    Pg = P if p_global is None else int(p_global)
    dl = None
    rows = None
    n_rows = 0
    if want_dlogits or dl_rows is not None:
        if dl_rows is not None:
            rows = np.ascontiguousarray(dl_rows, dtype=np.int64).reshape(-1)
            n_rows = rows.size
        else:
            n_rows = B * T
        dl = np.zeros((n_rows, V), np.float64)
    S = np.zeros(B, np.float64)
    z = np.zeros(P, np.float64)
    stats = np.zeros(10, np.float64)
    status = np.zeros(1, np.uint32)
    rs = np.zeros((B, T), np.float64) if unscaled else None
    args = [_ptr(a), dt, B, T, V, sb, st, _ptr(ref), _ptr(tok), _ptr(msk), _ptr(pr), P, Pg,
            float(np.float32(beta)), float(np.float32(inv_temperature)), _ptr(dl), _ptr(rows),
            n_rows]
    if unscaled:
        rc = lib().orc_online_dpo_loss_fwd_bwd_unscaled(
            *args, _ptr(rs), _ptr(S), _ptr(z), _ptr(stats), _ptr(status), int(n_threads))
    else:
        rc = lib().orc_online_dpo_loss_fwd_bwd(
            *args, _ptr(S), _ptr(z), _ptr(stats), _ptr(status), int(n_threads))
    if rc:
        raise ValueError("orc_online_dpo_loss_fwd_bwd: invalid argument")
    if dl is not None and dl_rows is None:
        dl = dl.reshape(B, T, V)
    return dict(seq_logp=S, z=z, stats=stats, status=int(status[0]), dlogits=dl, row_scale=rs)


PG_KINDS = {"rloo": 0, "copg": 1, "prox_rloo": 2, "sft": 3}


def pg_loss_fwd_bwd(logits, tokens, mask, kind, rewards, old_logp=None, clip_eps=0.2,
                    pair_rows=None, p_global=None, inv_temperature=1.0, want_dlogits=False,
                    dl_rows=None, n_threads=1):
    """Coefficient-variant losses (App B): returns dict(seq_logp[B], stats[10], status,
    dlogits[n, V] or None).  rewards[B] and old_logp[B] are per sequence."""
    a, dt, sb, st = _logits_args(logits)
    B, T, V = a.shape
    tok = np.ascontiguousarray(tokens, dtype=np.int32).reshape(B, T)
    msk = np.ascontiguousarray(mask, dtype=np.uint8).reshape(B, T)
    rew = np.ascontiguousarray(rewards, dtype=np.float32).reshape(B)
    old = None if old_logp is None else np.ascontiguousarray(old_logp, dtype=np.float32).reshape(B)
    pr = None if pair_rows is None else np.ascontiguousarray(pair_rows, dtype=np.int32).reshape(-1, 2)
    P = B // 2 if pr is None else pr.shape[0]
    Pg = P if p_global is None else int(p_global)
    dl, rows, n_rows = None, None, 0
    if want_dlogits or dl_rows is not None:
        if dl_rows is not None:
            rows = np.ascontiguousarray(dl_rows, dtype=np.int64).reshape(-1)
            n_rows = rows.size
        else:
            n_rows = B * T
        dl = np.zeros((n_rows, V), np.float64)
    S = np.zeros(B, np.float64)
    stats = np.zeros(10, np.float64)
    status = np.zeros(1, np.uint32)
    rc = lib().orc_pg_loss_fwd_bwd(
        _ptr(a), dt, B, T, V, sb, st, _ptr(tok), _ptr(msk), _ptr(pr), P, Pg, PG_KINDS[kind],
        _ptr(rew), _ptr(old), float(np.float32(clip_eps)), float(np.float32(inv_temperature)),
        _ptr(dl), _ptr(rows), n_rows, _ptr(S), _ptr(stats), _ptr(status), int(n_threads))
    if rc:
        raise ValueError("orc_pg_loss_fwd_bwd: invalid argument")
    if dl is not None and dl_rows is None:
        dl = dl.reshape(B, T, V)
    return dict(seq_logp=S, stats=stats, status=int(status[0]), dlogits=dl)


def lmhead_seq_logprobs(hidden, weight, tokens, mask, inv_temperature=1.0, n_threads=1):
    """NEXT-2: sequence log-probs from the LM head.  The logits are the LM
    head's definition, logits[b, t, v] = sum_i hidden[b, t, i] * weight[v, i], formed in fp64
    by a library matmul (hidden and weight hold bf16-exact values, so the fp64 products and
    sums are exact up to fp64 rounding); the log-softmax, gather and masked sum are
    seq_logprobs' (Sec 2.1).  Returns seq_logprobs' dict."""
    h = np.asarray(hidden, dtype=np.float64)
    w = np.asarray(weight, dtype=np.float64)
    if h.ndim != 3 or w.ndim != 2 or h.shape[2] != w.shape[1]:
        raise ValueError("hidden must be [B, T, d] and weight [V, d]")
    B, T, d = h.shape
    logits = (h.reshape(B * T, d) @ w.T).reshape(B, T, w.shape[0])
    return seq_logprobs(np.ascontiguousarray(logits), tokens, mask, inv_temperature, n_threads)


def lmhead_dpo_grad(hidden, weight, ref_logp, tokens, mask, beta, pair_rows=None,
                    p_global=None, inv_temperature=1.0, n_threads=1):
    """NEXT-2 backward oracle: gradients of the Online-DPO loss (online_dpo_loss_fwd_bwd on the
    head's fp64 logits) with respect to the LM head's input and weight, by the chain rule
    written out: G = row_scale * (softmax(invT * logits) - onehot) (row_scale = coef_b * mask
    from the unscaled loss oracle), dhidden = G @ weight, dweight = G.T @ hidden.  Returns
    dict(dhidden [B, T, d], dweight [V, d], row_scale, loss)."""
    h = np.asarray(hidden, dtype=np.float64)
    w = np.asarray(weight, dtype=np.float64)
    B, T, d = h.shape
    V = w.shape[0]
    logits = np.ascontiguousarray((h.reshape(B * T, d) @ w.T).reshape(B, T, V))
    o = online_dpo_loss_fwd_bwd(logits, ref_logp, tokens, mask, beta, pair_rows=pair_rows,
                                p_global=p_global, inv_temperature=inv_temperature,
                                n_threads=n_threads, unscaled=True)
    it = float(np.float32(inv_temperature))
    x = it * logits.reshape(B * T, V)
    x = x - x.max(axis=1, keepdims=True)
    p = np.exp(x)
    p /= p.sum(axis=1, keepdims=True)
    tok = np.asarray(tokens, dtype=np.int64).reshape(-1)
    p[np.arange(B * T), tok] -= 1.0
    G = o["row_scale"].reshape(B * T, 1) * p
    return dict(dhidden=(G @ w).reshape(B, T, d), dweight=G.T @ h.reshape(B * T, d),
                row_scale=o["row_scale"], loss=o["stats"][1], G=G)


def to_bf16_bits(x) -> np.ndarray:
    """Round float values to bf16 (round-to-nearest-even) and return the uint16 bits.

    Test helper for building BF16 oracle inputs; uses torch's CPU conversion."""
    import torch
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16)
    return t.view(torch.int16).numpy().view(np.uint16)


def bf16_bits_to_f64(bits) -> np.ndarray:
    b = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
    return b.view(np.float32).astype(np.float64)
