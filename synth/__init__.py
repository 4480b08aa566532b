"""Seeded synthetic-input generator shared by tests, bench and smoke.

This module holds NONE of the method's arithmetic (no softmax, no log-prob, no
loss): it only draws the inputs of the Online-DPO learner step from an
integer-only counter hash, so that the host (numpy, here) and the device
(``synth/synth.cu``, a separate CUDA twin) produce bit-identical data keyed by
GLOBAL indices.  Both the CPU oracle and the CUDA path consume what it draws;
neither imports the other.

Recipe (SURVEY.md §8(d) "Synthetic inputs"):

* hash        h(seed, stream, i) = splitmix64(splitmix64(seed*256 + stream) ^ i)
* logits      x[g, v] = int8(h(seed, S_LOGITS(+1 for ref), g*V + v) & 0xff) / 64
              -> a 1/64 grid on [-2, 2), exact in bf16 and fp32.
              "peaked" regime: x[g, tok[g]] = A (default 14.0, bf16-exact), which
              gives per-token log-probs of -0.05..-0.18, i.e. the paper's KL-proxy
              perplexity range 1.068-1.092.
* tokens      tok[g] = h(seed, S_TOKENS, g) % V
* masks       dense, or prefix with L_b = 1 + h(seed, S_MASK, b) % (2*Lbar - 1)
* rewards     RM-like grid ((h % 4096) - 2048) / 256 in [-8, 8)
              or verifier rewards h & 1 in {0, 1}
* has_eos     (h(seed, S_EOS, p*K + k) % 32) != 0  (~3% truncated completions)
* LM head     (NEXT-2) hidden[g, i] = ((h(seed, S_HIDDEN, g*d + i) % 64) - 32) / 32 and
              W[v, i] = ((h(seed, S_WEIGHT, v*d + i) % 64) - 32) / 256: dyadic grids exact in
              bf16, so hidden @ W.T is exact in fp64; logits have std ~ 0.04 sqrt(d)
              (2.1 at the Pythia-2.8B width d = 2560)
"""
from __future__ import annotations

import numpy as np

S_LOGITS = 1
S_LOGITS_REF = 2
S_TOKENS = 3
S_MASK = 4
S_REWARD = 5
S_EOS = 6
S_DELTA = 7
S_PERM = 8
S_SPLIT = 9
S_HIDDEN = 10
S_WEIGHT = 11

_G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(x):
    """splitmix64 finaliser on a uint64 array (wrapping arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + _G
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def stream_key(seed: int, stream: int) -> np.uint64:
    return splitmix64(np.array([(seed * 256 + stream) & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))[0]


def hash_u64(seed: int, stream: int, idx) -> np.ndarray:
    """h(seed, stream, idx) for an integer array of global indices."""
    idx = np.asarray(idx, dtype=np.uint64)
    return splitmix64(idx ^ stream_key(seed, stream))


def logits_rows(seed: int, rows_global, V: int, tokens=None, peak: float | None = 14.0,
                ref: bool = False) -> np.ndarray:
    """Logit rows [len(rows_global), V] as float64 (values exact in bf16/fp32)."""
    rows = np.asarray(rows_global, dtype=np.uint64).reshape(-1)
    stream = S_LOGITS_REF if ref else S_LOGITS
    out = np.empty((rows.size, V), dtype=np.float64)
    v = np.arange(V, dtype=np.uint64)
    key = stream_key(seed, stream)
    # chunk to bound the uint64 temporaries
    chunk = max(1, (1 << 22) // max(V, 1))
    for r0 in range(0, rows.size, chunk):
        rr = rows[r0:r0 + chunk]
        with np.errstate(over="ignore"):
            idx = rr[:, None] * np.uint64(V) + v[None, :]
        h = splitmix64(idx ^ key)
        b = (h & np.uint64(0xFF)).astype(np.uint8).view(np.int8)
        out[r0:r0 + chunk] = b.astype(np.float64) / 64.0
    if peak is not None and tokens is not None:
        tok = np.asarray(tokens, dtype=np.int64).reshape(-1)
        ok = (tok >= 0) & (tok < V)
        out[np.nonzero(ok)[0], tok[ok]] = peak
    return out


def tokens_rows(seed: int, rows_global, V: int) -> np.ndarray:
    h = hash_u64(seed, S_TOKENS, rows_global)
    return (h % np.uint64(V)).astype(np.int32)


def prefix_lengths(seed: int, seqs_global, T: int, lbar: int) -> np.ndarray:
    h = hash_u64(seed, S_MASK, seqs_global)
    L = 1 + (h % np.uint64(2 * lbar - 1)).astype(np.int64)
    return np.minimum(L, T)


def mask_for(seed: int, seqs_global, T: int, kind: str = "dense", lbar: int | None = None) -> np.ndarray:
    seqs = np.asarray(seqs_global, dtype=np.int64).reshape(-1)
    if kind == "dense":
        return np.ones((seqs.size, T), dtype=np.uint8)
    if kind == "prefix":
        L = prefix_lengths(seed, seqs, T, lbar if lbar else max(1, T // 2))
        return (np.arange(T)[None, :] < L[:, None]).astype(np.uint8)
    raise ValueError(kind)


def rewards_for(seed: int, P: int, K: int, p0: int = 0, kind: str = "rm") -> np.ndarray:
    idx = (np.arange(P, dtype=np.int64)[:, None] + p0) * K + np.arange(K, dtype=np.int64)[None, :]
    h = hash_u64(seed, S_REWARD, idx.reshape(-1)).reshape(P, K)
    if kind == "rm":
        return (((h % np.uint64(4096)).astype(np.int64) - 2048) / 256.0).astype(np.float32)
    if kind == "verifier":
        return (h & np.uint64(1)).astype(np.float32)
    raise ValueError(kind)


def has_eos_for(seed: int, P: int, K: int, p0: int = 0) -> np.ndarray:
    idx = (np.arange(P, dtype=np.int64)[:, None] + p0) * K + np.arange(K, dtype=np.int64)[None, :]
    h = hash_u64(seed, S_EOS, idx.reshape(-1)).reshape(P, K)
    return ((h % np.uint64(32)) != 0).astype(np.uint8)


def uniform_u32(seed: int, stream: int, idx) -> np.ndarray:
    return (hash_u64(seed, stream, idx) >> np.uint64(32)).astype(np.uint32)


def permutation(seed: int, n: int, stream: int = S_PERM) -> np.ndarray:
    """A seeded permutation of range(n) (sort by hash)."""
    h = hash_u64(seed, stream, np.arange(n))
    return np.argsort(h, kind="stable").astype(np.int32)


# ----------------------------------------------------------------------------- device twin
import ctypes as _C
import os as _os
import subprocess as _sp

_HERE = _os.path.dirname(_os.path.abspath(__file__))
SYNTH_LIB = _os.path.join(_HERE, "libsynth.so")
_slib = None


def build_device(force: bool = False) -> str:
    src = _os.path.join(_HERE, "synth.cu")
    if force or not _os.path.exists(SYNTH_LIB) or _os.path.getmtime(SYNTH_LIB) < _os.path.getmtime(src):
        _sp.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                        "-Xcompiler", "-fPIC", "-shared", "-o", SYNTH_LIB, src])
    return SYNTH_LIB


def _dev_lib():
    global _slib
    if _slib is None:
        if not _os.path.exists(SYNTH_LIB):
            build_device()
        L = _C.CDLL(SYNTH_LIB)
        L.synth_fill_logits.argtypes = [_C.c_void_p, _C.c_int, _C.c_int64, _C.c_int64, _C.c_int64,
                                        _C.c_int64, _C.c_int64, _C.c_uint64, _C.c_int, _C.c_int64,
                                        _C.c_void_p, _C.c_float, _C.c_int, _C.c_void_p]
        L.synth_fill_logits.restype = _C.c_int
        L.synth_read_probe.argtypes = [_C.c_void_p, _C.c_int64, _C.c_void_p, _C.c_int, _C.c_void_p]
        L.synth_read_probe.restype = _C.c_int
        L.synth_stream_key.argtypes = [_C.c_uint64, _C.c_int]
        L.synth_stream_key.restype = _C.c_uint64
        _slib = L
    return _slib


def fill_logits_device(x, seed: int, row0: int = 0, tokens=None, peak: float | None = 14.0,
                       ref: bool = False) -> None:
    """Fill a CUDA tensor x[B, T, V] (f32 or bf16, last dim contiguous) with the same values
    logits_rows() produces for global rows row0 + b*T + t.  tokens: CUDA int32 [B, T] or None."""
    import torch
    assert x.is_cuda and x.dim() == 3 and x.stride(2) == 1
    dt = {torch.float32: 0, torch.bfloat16: 1}[x.dtype]
    B, T, V = x.shape
    tk = None
    if tokens is not None and peak is not None:
        assert tokens.is_cuda and tokens.dtype == torch.int32 and tokens.is_contiguous()
        tk = tokens.data_ptr()
    rc = _dev_lib().synth_fill_logits(
        x.data_ptr(), dt, B, T, V, x.stride(0), x.stride(1), seed,
        S_LOGITS_REF if ref else S_LOGITS, row0, tk, float(peak if peak is not None else 0.0),
        1 if tk is not None else 0, torch.cuda.current_stream().cuda_stream)
    if rc:
        raise RuntimeError(f"synth_fill_logits failed ({rc})")


def read_probe(x, blocks: int) -> None:
    """bench.py ceiling probe: stream x's bytes once (read only) on the current stream."""
    import torch
    out = torch.zeros(1, dtype=torch.int32, device=x.device)
    rc = _dev_lib().synth_read_probe(x.data_ptr(), x.numel() * x.element_size(), out.data_ptr(),
                                     int(blocks), torch.cuda.current_stream().cuda_stream)
    if rc:
        raise RuntimeError(f"synth_read_probe failed ({rc})")


def lmhead_inputs(seed: int, rows_global, d: int, V: int, v_rows=None):
    """NEXT-2 inputs: hidden [len(rows_global), d] and W [V, d] (or the rows v_rows of W) as
    float64 arrays whose values are exact in bf16 (see the recipe above)."""
    rows_global = np.asarray(rows_global, dtype=np.uint64)
    i = np.arange(d, dtype=np.uint64)
    h = hash_u64(seed, S_HIDDEN, rows_global[:, None] * np.uint64(d) + i[None, :])
    hidden = ((h % np.uint64(64)).astype(np.int64) - 32).astype(np.float64) / 32.0
    vr = np.arange(V, dtype=np.uint64) if v_rows is None else np.asarray(v_rows, dtype=np.uint64)
    w = hash_u64(seed, S_WEIGHT, vr[:, None] * np.uint64(d) + i[None, :])
    weight = ((w % np.uint64(64)).astype(np.int64) - 32).astype(np.float64) / 256.0
    return hidden, weight

