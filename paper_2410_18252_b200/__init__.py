"""paper_2410_18252_b200 -- B200-native Online-DPO learner hot path (arXiv 2410.18252).

Thin Python binding over the C-ABI library ``libodpo.so`` (declared in
``include/odpo.h``).  This module only marshals arguments: every step of the path
runs in the library's sm_100a kernels.  PyTorch supplies device memory, the
current CUDA stream and ``torch.distributed`` process groups.  There is no CPU
fallback: importing this package without the built library, or calling it with
CPU tensors, raises.

Calls (Sec 2.1):
  pair_select(rewards, has_eos, eos_penalty)
  seq_logprobs(logits, tokens, mask, inv_temperature)
  online_dpo_loss_fwd_bwd(policy_logits, ref_logp, tokens, mask, beta, ...)
  allreduce_stats(stats_buffer)   -- the batch-sharded NCCL stats reduction
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import torch

__all__ = ["pair_select", "seq_logprobs", "seq_ppl", "VPExchange", "vp_loss_step", "set_tracing", "online_dpo_loss_fwd_bwd", "allreduce_stats",
           "workspace_bytes", "LossOutput", "SelectOutput", "OdpoError", "lib_path",
           "STAT_NAMES", "SEL_NAMES", "FLAGS"]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libodpo.so")

STAT_NAMES = ["npairs", "loss", "ncorrect", "z_sum", "rchosen_sum", "rrej_sum",
              "schosen_sum", "srej_sum", "ntok_chosen", "ntok_rej"]
SEL_NAMES = ["margin_sum", "ndegen", "ntrunc"]
NSTATS, NSEL, STATS_BUF = 10, 3, 16
FLAGS = {"TOKEN_RANGE": 1, "NONFINITE_LOGIT": 2, "EMPTY_SEQ": 4, "NONFINITE_REWARD": 8,
         "DUP_ROW": 16, "DEGENERATE_PAIR": 32, "PAIR_RANGE": 64}
SCHEDULES = {"auto": 0, "fused": 1, "two_pass": 2, "wave": 3, "resident": 4, "psync": 5,
             "split": 6}
_DT = {torch.float32: 0, torch.bfloat16: 1}


class OdpoError(RuntimeError):
    pass


_TRACE = False


def set_tracing(enabled: bool) -> None:
    """NVTX ranges around every call of this module (SURVEY.md §5 tracing): each public call
    pushes a range named after it (e.g. "odpo.online_dpo_loss_fwd_bwd") for nsys / ncu
    --nvtx timelines.  Off by default (one flag test per call)."""
    global _TRACE
    _TRACE = bool(enabled)


def _traced(fn):
    import functools
    name = "odpo." + fn.__name__

    @functools.wraps(fn)
    def wrapper(*args, **kw):
        if not _TRACE:
            return fn(*args, **kw)
        torch.cuda.nvtx.range_push(name)
        try:
            return fn(*args, **kw)
        finally:
            torch.cuda.nvtx.range_pop()
    return wrapper


class _Opts(C.Structure):
    _fields_ = [("schedule", C.c_int32), ("lag_pairs", C.c_int32), ("ctas_per_sm", C.c_int32),
                ("launches", C.c_int32), ("exp2_split", C.c_int32), ("lookahead", C.c_int32),
                ("row_gap", C.c_int32), ("engine", C.c_int32)]


_lib = None


def lib_path() -> str:
    return LIB_PATH


def _L():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise OdpoError(f"libodpo.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        P, i64, i32, f32, sz = C.c_void_p, C.c_int64, C.c_int32, C.c_float, C.c_size_t
        L.odpo_pair_select.argtypes = [P, P, f32, i64, i32, P, P, P, P, P, P, P]
        L.odpo_seq_logprobs.argtypes = [P, C.c_int, i64, i64, i64, i64, i64, P, P, f32, P, P, P, P,
                                        P, sz, P]
        L.odpo_seq_ppl.argtypes = [P, C.c_int, i64, i64, i64, i64, i64, P, P, f32, P, P, P, P, P,
                                   sz, P]
        L.odpo_seq_ppl.restype = C.c_int
        L.odpo_online_dpo_loss_fwd_bwd.argtypes = [P, C.c_int, i64, i64, i64, i64, i64, P, P, P, P,
                                                   i64, i64, f32, f32, P, i64, i64, P, P, P, P, P,
                                                   sz, P]
        L.odpo_online_dpo_loss_fwd_bwd_ex.argtypes = (L.odpo_online_dpo_loss_fwd_bwd.argtypes[:-1]
                                                      + [C.POINTER(_Opts), P])
        L.odpo_online_dpo_loss_fwd_bwd_unscaled.argtypes = [
            P, C.c_int, i64, i64, i64, i64, i64, P, P, P, P, i64, i64, f32, f32, P, i64, i64, P, P,
            P, P, P, P, sz, C.POINTER(_Opts), P]
        L.odpo_vp_row_partials.argtypes = [P, C.c_int, i64, i64, i64, i64, i64, i64, i64, P, P,
                                           f32, P, P, P, sz, P]
        L.odpo_vp_loss_fwd_bwd.argtypes = [P, i32, P, C.c_int, i64, i64, i64, i64, i64, i64, i64,
                                           P, P, P, P, i64, i64, f32, f32, P, i64, i64, P, P, P,
                                           P, C.c_uint32, P, P, sz, P]
        L.odpo_vp_row_partials_put.argtypes = [P, C.c_int, i64, i64, i64, i64, i64, i64, i64, P,
                                               P, f32, C.POINTER(P), C.POINTER(P), P, i32, i32,
                                               C.c_uint32, P, P]
        L.odpo_vp_row_partials_put.restype = C.c_int
        L.odpo_stats_put.argtypes = [P, C.POINTER(P), C.POINTER(P), i32, i32, C.c_uint32, P]
        L.odpo_stats_put.restype = C.c_int
        L.odpo_stats_sum.argtypes = [P, P, i32, C.c_uint32, P, P]
        L.odpo_stats_sum.restype = C.c_int
        L.odpo_vp_row_partials.restype = C.c_int
        L.odpo_vp_loss_fwd_bwd.restype = C.c_int
        L.odpo_gather_pairs.argtypes = [P, i64, i64, i64, P, P, P, P, P, P, P, P]
        L.odpo_gather_pairs.restype = C.c_int
        L.odpo_pg_loss_fwd_bwd.argtypes = [
            P, C.c_int, i64, i64, i64, i64, i64, P, P, P, i64, i64, i32, P, P, f32, f32, P, i64,
            i64, P, P, P, P, sz, C.POINTER(_Opts), P]
        for f in (L.odpo_pair_select, L.odpo_seq_logprobs, L.odpo_online_dpo_loss_fwd_bwd,
                  L.odpo_online_dpo_loss_fwd_bwd_ex, L.odpo_online_dpo_loss_fwd_bwd_unscaled,
                  L.odpo_pg_loss_fwd_bwd):
            f.restype = C.c_int
        L.odpo_lmhead_seq_logprobs.argtypes = [P, P, i64, i64, i64, i64, P, P, f32, P, P, P, P,
                                               P, sz, P]
        L.odpo_lmhead_seq_logprobs.restype = C.c_int
        L.odpo_lmhead_workspace_bytes.argtypes = [i64, i64, i64]
        L.odpo_lmhead_workspace_bytes.restype = sz
        L.odpo_online_dpo_loss_from_token_logp.argtypes = [P, i64, i64, P, P, P, i64, i64, f32,
                                                           f32, P, P, P, P, P, P, sz, P]
        L.odpo_online_dpo_loss_from_token_logp.restype = C.c_int
        L.odpo_lmhead_grad_scratch_bytes.argtypes = [i64, i64, i64]
        L.odpo_lmhead_grad_scratch_bytes.restype = sz
        L.odpo_lmhead_grad.argtypes = [P, P, i64, i64, i64, P, P, P, f32, P, P, P, sz, i64, P]
        L.odpo_lmhead_grad.restype = C.c_int
        L.odpo_lmhead_dpo_step_scratch_bytes.argtypes = [i64, i64, i64]
        L.odpo_lmhead_dpo_step_scratch_bytes.restype = sz
        L.odpo_lmhead_dpo_step.argtypes = [P, P, i64, i64, i64, i64, P, P, P, i64, f32, f32, P, P,
                                           P, P, P, P, P, sz, i64, P]
        L.odpo_lmhead_dpo_step.restype = C.c_int
        L.odpo_workspace_bytes.argtypes = [i64, i64, i64]
        L.odpo_workspace_bytes.restype = sz
        L.odpo_status_string.argtypes = [C.c_int]
        L.odpo_status_string.restype = C.c_char_p
        L.odpo_version.restype = C.c_char_p
        _lib = L
    return _lib


def _check(rc: int, what: str):
    if rc != 0:
        raise OdpoError(f"{what}: {_L().odpo_status_string(rc).decode()} (code {rc})")


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _dev(t, name, dtype=None):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise OdpoError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if dtype is not None and t.dtype != dtype:
        raise OdpoError(f"{name} must be {dtype}, got {t.dtype}")
    return t


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def workspace_bytes(B: int, T: int, P: int) -> int:
    return int(_L().odpo_workspace_bytes(B, T, P))


_ws_cache: dict = {}


def _workspace(device, nbytes: int):
    """Scratch for one call, cached per (device, stream): calls on one stream are ordered,
    so they may share a buffer; calls on different streams never do (each stream's buffer
    comes from the caching allocator's pool of that stream, so a replaced buffer is reused
    only after the work queued on its stream)."""
    dev = device.index if device.index is not None else torch.cuda.current_device()
    key = (dev, torch.cuda.current_stream(dev).cuda_stream)
    buf = _ws_cache.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        _ws_cache[key] = buf
    return buf


def _tokmask(tokens, mask, B, T):
    tokens = _dev(tokens, "tokens", torch.int32).contiguous()
    mask = _dev(mask, "mask", torch.uint8).contiguous()
    if tokens.numel() != B * T or mask.numel() != B * T:
        raise OdpoError(f"tokens and mask must be [B, T] = [{B}, {T}]")
    return tokens, mask


def _status(status, dev):
    if status is None:
        return torch.zeros(1, dtype=torch.int32, device=dev)
    _dev(status, "status", torch.int32)
    if status.numel() < 1:
        raise OdpoError("status must hold one int32")
    return status


def _stats(stats, dev, n=16):
    if stats is None:
        return torch.zeros(n, dtype=torch.float64, device=dev)
    _dev(stats, "stats", torch.float64)
    if not stats.is_contiguous() or stats.numel() < NSTATS:
        raise OdpoError(f"stats must be a contiguous float64 buffer of >= {NSTATS} doubles")
    return stats


def _per_seq(x, name, B):
    x = _dev(x, name, torch.float32).contiguous()
    if x.numel() != B:
        raise OdpoError(f"{name} must hold one float per sequence ({B})")
    return x


def _pairs(pair_rows, B):
    if pair_rows is None:
        if B % 2:
            raise OdpoError("pair_rows=None needs an even number of sequences (rows 2p, 2p+1)")
        return None, B // 2
    pair_rows = _dev(pair_rows, "pair_rows", torch.int32).contiguous()
    if pair_rows.dim() != 2 or pair_rows.shape[1] != 2:
        raise OdpoError("pair_rows must be [P, 2]")
    return pair_rows, pair_rows.shape[0]


def _out_rows(out, like, name):
    """A caller-supplied [B, T, V] output: same shape and dtype as the logits, contiguous V."""
    _dev(out, name, like.dtype)
    if tuple(out.shape) != tuple(like.shape) or out.stride(2) != 1:
        raise OdpoError(f"{name} must be [B, T, V] = {tuple(like.shape)} with a contiguous last "
                        f"dimension")
    return out


@dataclass
class SelectOutput:
    chosen: torch.Tensor
    rejected: torch.Tensor
    pair_rows: torch.Tensor
    reward_margin: torch.Tensor
    sel_stats: torch.Tensor
    status: torch.Tensor


@_traced
def pair_select(rewards: torch.Tensor, has_eos: torch.Tensor | None = None, eos_penalty: float = -1.0,
                status: torch.Tensor | None = None, sel_stats: torch.Tensor | None = None) -> SelectOutput:
    """Reward-ranked pair selection (EOS penalty PAPER.md:434-435)."""
    _dev(rewards, "rewards", torch.float32)
    rewards = rewards.contiguous()
    P, K = rewards.shape
    dev = rewards.device
    if has_eos is not None:
        has_eos = _dev(has_eos, "has_eos", torch.uint8).contiguous()
    chosen = torch.empty(P, dtype=torch.int32, device=dev)
    rejected = torch.empty(P, dtype=torch.int32, device=dev)
    pair_rows = torch.empty((P, 2), dtype=torch.int32, device=dev)
    margin = torch.empty(P, dtype=torch.float32, device=dev)
    if sel_stats is None:
        sel_stats = torch.zeros(NSEL, dtype=torch.float64, device=dev)
    status = _status(status, dev)
    _check(_L().odpo_pair_select(_p(rewards), _p(has_eos), float(eos_penalty), P, K, _p(chosen),
                                 _p(rejected), _p(pair_rows), _p(margin), _p(sel_stats), _p(status),
                                 _stream()), "odpo_pair_select")
    return SelectOutput(chosen, rejected, pair_rows, margin, sel_stats, status)


@_traced
def gather_pairs(pair_rows: torch.Tensor, tokens: torch.Tensor, mask: torch.Tensor,
                 ref_logp: torch.Tensor | None = None, status: torch.Tensor | None = None):
    """Selected completions in pair order: returns (tokens[2P, T],
    mask[2P, T], ref_logp[2P] or None) for a loss call with pair_rows=None."""
    pair_rows = _dev(pair_rows, "pair_rows", torch.int32).contiguous()
    tokens = _dev(tokens, "tokens", torch.int32).contiguous()
    mask = _dev(mask, "mask", torch.uint8).contiguous()
    P = pair_rows.shape[0]
    n_src, T = tokens.shape
    dev = tokens.device
    tok_o = torch.empty((2 * P, T), dtype=torch.int32, device=dev)
    mask_o = torch.empty((2 * P, T), dtype=torch.uint8, device=dev)
    ref_o = None
    if ref_logp is not None:
        ref_logp = _dev(ref_logp, "ref_logp", torch.float32).contiguous()
        ref_o = torch.empty(2 * P, dtype=torch.float32, device=dev)
    _check(_L().odpo_gather_pairs(_p(pair_rows), P, n_src, T, _p(tokens), _p(mask), _p(ref_logp),
                                  _p(tok_o), _p(mask_o), _p(ref_o), _p(status), _stream()),
           "odpo_gather_pairs")
    return tok_o, mask_o, ref_o


def _logits_meta(x: torch.Tensor, name="logits"):
    _dev(x, name)
    if x.dtype not in _DT:
        raise OdpoError(f"{name} dtype must be float32 or bfloat16")
    if x.dim() != 3 or x.stride(2) != 1:
        raise OdpoError(f"{name} must be [B, T, V] with a contiguous last dimension")
    return _DT[x.dtype], x.shape[0], x.shape[1], x.shape[2], x.stride(0), x.stride(1)


def _rows_like(x: torch.Tensor) -> torch.Tensor:
    """An output [B, T, V] with x's dtype whose row stride is padded to 16 bytes (the C ABI's
    alignment contract), so a default output is valid for every valid input."""
    B, T, V = x.shape
    es = x.element_size()
    vp = -(-V * es // 16) * 16 // es
    return torch.empty((B, T, vp), dtype=x.dtype, device=x.device)[:, :, :V]


@_traced
def seq_logprobs(logits: torch.Tensor, tokens: torch.Tensor, mask: torch.Tensor,
                 inv_temperature: float = 1.0, per_token: bool = False,
                 status: torch.Tensor | None = None):
    """log pi(y|x) per sequence.  Returns seq_logp[B] (and tok_logp, row_lse
    [B, T] when per_token=True)."""
    dt, B, T, V, sb, st = _logits_meta(logits)
    tokens, mask = _tokmask(tokens, mask, B, T)
    dev = logits.device
    seq = torch.empty(B, dtype=torch.float32, device=dev)
    tok = lse = None
    if per_token:
        tok = torch.empty((B, T), dtype=torch.float32, device=dev)
        lse = torch.empty((B, T), dtype=torch.float32, device=dev)
    status = _status(status, dev)
    nb = workspace_bytes(B, T, B // 2 + 1)
    ws = _workspace(dev, nb)
    _check(_L().odpo_seq_logprobs(_p(logits), dt, B, T, V, sb, st, _p(tokens), _p(mask),
                                  float(inv_temperature), _p(seq), _p(tok), _p(lse), _p(status),
                                  _p(ws), ws.numel(), _stream()), "odpo_seq_logprobs")
    if per_token:
        return seq, tok, lse, status
    return seq


@_traced
def seq_ppl(logits: torch.Tensor, tokens: torch.Tensor, mask: torch.Tensor,
            inv_temperature: float = 1.0, status: torch.Tensor | None = None):
    """KL proxy: with the reference model's logits, the per-completion
    perplexity exp(-S_b / n_b).  Returns (ppl [B] f32, ppl_stats [4] f64 = (#non-empty,
    sum ppl, sum S, sum n), seq_logp [B], status)."""
    dt, B, T, V, sb, st = _logits_meta(logits)
    tokens, mask = _tokmask(tokens, mask, B, T)
    dev = logits.device
    seq = torch.empty(B, dtype=torch.float32, device=dev)
    ppl = torch.empty(B, dtype=torch.float32, device=dev)
    ps = torch.zeros(4, dtype=torch.float64, device=dev)
    status = _status(status, dev)
    ws = _workspace(dev, workspace_bytes(B, T, B // 2 + 1))
    _check(_L().odpo_seq_ppl(_p(logits), dt, B, T, V, sb, st, _p(tokens), _p(mask),
                             float(inv_temperature), _p(seq), _p(ppl), _p(ps), _p(status),
                             _p(ws), ws.numel(), _stream()), "odpo_seq_ppl")
    return ppl, ps, seq, status


@_traced
def lmhead_seq_logprobs(hidden: torch.Tensor, weight: torch.Tensor, tokens: torch.Tensor,
                        mask: torch.Tensor, inv_temperature: float = 1.0,
                        status: torch.Tensor | None = None):
    """log pi(y|x) per sequence straight from the LM head (forward):
    hidden [B, T, d] bf16, weight [V, d] bf16 (both contiguous, d % 64 == 0); the logits
    hidden @ weight.T * invT are formed tile by tile in tensor memory (tcgen05) and never
    written.  Returns (seq_logp [B], tok_logp [B, T], row_lse [B, T], status)."""
    hidden = _dev(hidden, "hidden", torch.bfloat16)
    weight = _dev(weight, "weight", torch.bfloat16)
    if hidden.dim() != 3 or weight.dim() != 2 or hidden.shape[2] != weight.shape[1]:
        raise ValueError("hidden must be [B, T, d] and weight [V, d]")
    if not (hidden.is_contiguous() and weight.is_contiguous()):
        raise ValueError("hidden and weight must be contiguous")
    B, T, d = hidden.shape
    V = weight.shape[0]
    tokens, mask = _tokmask(tokens, mask, B, T)
    dev = hidden.device
    seq = torch.empty(B, dtype=torch.float32, device=dev)
    tok = torch.empty((B, T), dtype=torch.float32, device=dev)
    lse = torch.empty((B, T), dtype=torch.float32, device=dev)
    status = _status(status, dev)
    nb = _L().odpo_lmhead_workspace_bytes(B, T, V)
    ws = _workspace(dev, nb)
    _check(_L().odpo_lmhead_seq_logprobs(_p(hidden), _p(weight), B, T, d, V, _p(tokens), _p(mask),
                                         float(inv_temperature), _p(tok), _p(lse), _p(seq),
                                         _p(status), _p(ws), ws.numel(), _stream()),
           "odpo_lmhead_seq_logprobs")
    return seq, tok, lse, status


@_traced
def lmhead_online_dpo_loss_fwd(hidden: torch.Tensor, weight: torch.Tensor,
                               ref_logp: torch.Tensor, tokens: torch.Tensor, mask: torch.Tensor,
                               beta: float, pair_rows: torch.Tensor | None = None,
                               p_global: int | None = None, inv_temperature: float = 1.0):
    """NEXT-2 forward: the Online-DPO loss, statistics and per-row gradient scale straight from
    the policy's LM head (hidden [B, T, d] bf16, weight [V, d] bf16), logits never stored.
    Returns LossOutput with dlogits = None and row_scale [B, T] = coef_b * mask."""
    _, tok_logp, row_lse, status = lmhead_seq_logprobs(hidden, weight, tokens, mask,
                                                       inv_temperature)
    B, T = tok_logp.shape
    dev = hidden.device
    ref_logp = _per_seq(ref_logp, "ref_logp", B)
    mask = _dev(mask, "mask", torch.uint8).contiguous()
    pair_rows, P = _pairs(pair_rows, B)
    Pg = P if p_global is None else int(p_global)
    seq = torch.empty(B, dtype=torch.float32, device=dev)
    z = torch.empty(max(P, 1), dtype=torch.float32, device=dev)
    stats = torch.zeros(STATS_BUF, dtype=torch.float64, device=dev)
    row_scale = torch.empty((B, T), dtype=torch.float32, device=dev)
    ws = _workspace(dev, workspace_bytes(B, T, P))
    _check(_L().odpo_online_dpo_loss_from_token_logp(
        _p(tok_logp), B, T, _p(ref_logp), _p(mask), _p(pair_rows), P, Pg, float(beta),
        float(inv_temperature), _p(seq), _p(z), _p(stats), _p(row_scale), _p(status), _p(ws),
        ws.numel(), _stream()), "odpo_online_dpo_loss_from_token_logp")
    return LossOutput(stats=stats, dlogits=None, seq_logp=seq, z=z, status=status, launches=5,
                      row_scale=row_scale, row_lse=row_lse)


@_traced
def lmhead_grad(hidden: torch.Tensor, weight: torch.Tensor, tokens: torch.Tensor,
                row_lse: torch.Tensor, row_scale: torch.Tensor, inv_temperature: float = 1.0,
                chunk_rows: int | None = None):
    """NEXT-2 backward: (dhidden fp32 [B, T, d], dweight fp32 [V, d]) of the loss whose logit
    gradient is row_scale * (softmax - onehot); logits recomputed chunk by chunk on tcgen05,
    G and G^T written to a bf16 scratch of chunk_rows rows, then the library's own tcgen05
    GEMMs dhidden = G W and dweight += G^T H (no cuBLAS)."""
    hidden = _dev(hidden, "hidden", torch.bfloat16)
    weight = _dev(weight, "weight", torch.bfloat16)
    if not (hidden.is_contiguous() and weight.is_contiguous()):
        raise ValueError("hidden and weight must be contiguous")
    d = hidden.shape[-1]
    R = hidden.numel() // d
    V = weight.shape[0]
    tokens = _dev(tokens, "tokens", torch.int32).contiguous()
    row_lse = _dev(row_lse, "row_lse", torch.float32).contiguous()
    row_scale = _dev(row_scale, "row_scale", torch.float32).contiguous()
    if tokens.numel() != R or row_lse.numel() != R or row_scale.numel() != R:
        raise OdpoError(f"tokens, row_lse and row_scale must hold one value per row ({R})")
    dev = hidden.device
    dh = torch.empty(hidden.shape, dtype=torch.float32, device=dev)
    dw = torch.empty((V, d), dtype=torch.float32, device=dev)
    if chunk_rows is None:
        # whole waves of the dhidden GEMM: (chunk/256 row blocks) x (d/256 column blocks) tiles
        # a multiple of the CTA-pair count
        import math
        pairs = torch.cuda.get_device_properties(dev).multi_processor_count // 2
        nnb = -(-d // 256)
        chunk_rows = 256 * (pairs // math.gcd(pairs, nnb))
    cr = min(int(chunk_rows), R)
    cr = -(-cr // 256) * 256
    nb = _L().odpo_lmhead_grad_scratch_bytes(cr, d, V)
    scratch = torch.empty(max(nb, 256), dtype=torch.uint8, device=dev)
    _check(_L().odpo_lmhead_grad(_p(hidden), _p(weight), R, d, V, _p(tokens), _p(row_lse),
                                 _p(row_scale), float(inv_temperature), _p(dh), _p(dw),
                                 _p(scratch), scratch.numel(), cr, _stream()), "odpo_lmhead_grad")
    return dh, dw


@_traced
def lmhead_dpo_step(hidden: torch.Tensor, weight: torch.Tensor, ref_logp: torch.Tensor,
                    tokens: torch.Tensor, mask: torch.Tensor, beta: float,
                    p_global: int | None = None, inv_temperature: float = 1.0,
                    chunk_pairs: int | None = None, stats: torch.Tensor | None = None,
                    status: torch.Tensor | None = None):
    """NEXT-2 learner step in chunks of whole pairs (sequences (2p, 2p+1)): per chunk the logits
    in bf16 (library tcgen05 GEMM), the Online-DPO loss call in place, dhidden = dlogits W and
    dweight += dlogits^T hidden (library tcgen05 GEMMs).  Returns (LossOutput without dlogits,
    dhidden fp32 [B, T, d], dweight fp32 [V, d])."""
    hidden = _dev(hidden, "hidden", torch.bfloat16)
    weight = _dev(weight, "weight", torch.bfloat16)
    if hidden.dim() != 3 or weight.dim() != 2 or hidden.shape[2] != weight.shape[1]:
        raise OdpoError("hidden must be [B, T, d] and weight [V, d]")
    if not (hidden.is_contiguous() and weight.is_contiguous()):
        raise OdpoError("hidden and weight must be contiguous")
    B, T, d = hidden.shape
    V = weight.shape[0]
    if B % 2:
        raise OdpoError("the step takes the selected pairs as sequences (2p, 2p+1)")
    P = B // 2
    Pg = P if p_global is None else int(p_global)
    tokens, mask = _tokmask(tokens, mask, B, T)
    ref_logp = _per_seq(ref_logp, "ref_logp", B)
    dev = hidden.device
    if chunk_pairs is None:
        # at most ~1 GB of bf16 logits per chunk, and among those sizes the one whose dhidden
        # GEMM tiles ((rows/256) x (d/256)) fill the CTA-pair waves best
        cap = max(1, min(P, int((1 << 30) // max(1, 2 * T * V * 2))))
        pairs_sm = torch.cuda.get_device_properties(dev).multi_processor_count // 2
        nnb = -(-d // 256)

        def waste(cp):
            tiles = -(-(2 * cp * T) // 256) * nnb
            waves = -(-tiles // pairs_sm)
            nch = -(-P // cp)
            return (waves * pairs_sm - tiles) / (waves * pairs_sm) + 0.02 * nch
        chunk_pairs = min(range(max(1, cap // 2), cap + 1), key=lambda cp: (waste(cp), -cp))
    chunk_pairs = min(int(chunk_pairs), P)
    dh = torch.empty((B, T, d), dtype=torch.float32, device=dev)
    dw = torch.empty((V, d), dtype=torch.float32, device=dev)
    seq = torch.empty(B, dtype=torch.float32, device=dev)
    z = torch.empty(P, dtype=torch.float32, device=dev)
    stats = _stats(stats, dev)
    status = _status(status, dev)
    nb = _L().odpo_lmhead_dpo_step_scratch_bytes(chunk_pairs, T, V)
    scratch = torch.empty(max(nb, 256), dtype=torch.uint8, device=dev)
    _check(_L().odpo_lmhead_dpo_step(_p(hidden), _p(weight), P, T, d, V, _p(ref_logp), _p(tokens),
                                     _p(mask), Pg, float(beta), float(inv_temperature), _p(dh),
                                     _p(dw), _p(seq), _p(z), _p(stats), _p(status), _p(scratch),
                                     scratch.numel(), chunk_pairs, _stream()),
           "odpo_lmhead_dpo_step")
    return LossOutput(stats=stats, dlogits=None, seq_logp=seq, z=z, status=status,
                      launches=0), dh, dw


@dataclass
class LossOutput:
    stats: torch.Tensor       # fp64 [16]: loss stats [0,10), selection stats [10,13)
    dlogits: torch.Tensor
    seq_logp: torch.Tensor
    z: torch.Tensor
    status: torch.Tensor
    launches: int
    row_scale: torch.Tensor | None = None  # unscaled call: dlogits holds G, grad = row_scale * G
    row_lse: torch.Tensor | None = None    # LM-head loss forward: logsumexp per row (backward)

    def named(self) -> dict:
        s = self.stats.tolist()
        return {k: s[i] for i, k in enumerate(STAT_NAMES)}


@_traced
def online_dpo_loss_fwd_bwd(policy_logits: torch.Tensor, ref_logp: torch.Tensor,
                            tokens: torch.Tensor, mask: torch.Tensor, beta: float,
                            pair_rows: torch.Tensor | None = None, p_global: int | None = None,
                            inv_temperature: float = 1.0, inplace: bool = False,
                            dlogits: torch.Tensor | None = None, schedule: str = "auto",
                            lag_pairs: int = 0, ctas_per_sm: int = 0, exp2_split: int = -1,
                            lookahead: int = -1, engine: int = -1, row_gap: int = -1,
                            stats: torch.Tensor | None = None,
                            status: torch.Tensor | None = None) -> LossOutput:
    """Online DPO loss, statistics and dlogits in one call.

    stats: optional fp64 buffer of >= 10 doubles (the recommended 16-double buffer whose
    [10,13) holds pair_select's sel_stats); loss stats are written to stats[0:10]."""
    dt, B, T, V, sb, st = _logits_meta(policy_logits, "policy_logits")
    ref_logp = _per_seq(ref_logp, "ref_logp", B)
    tokens, mask = _tokmask(tokens, mask, B, T)
    dev = policy_logits.device
    pair_rows, P = _pairs(pair_rows, B)
    Pg = P if p_global is None else int(p_global)
    if inplace:
        dl = policy_logits
    elif dlogits is not None:
        dl = _out_rows(dlogits, policy_logits, "dlogits")
    else:
        dl = _rows_like(policy_logits)
    if dl.dim() != 3 or dl.stride(2) != 1:
        raise OdpoError("dlogits must be [B, T, V] with a contiguous last dimension")
    seq = torch.empty(B, dtype=torch.float32, device=dev)
    z = torch.empty(max(P, 1), dtype=torch.float32, device=dev)
    stats = _stats(stats, dev)
    status = _status(status, dev)
    nb = workspace_bytes(B, T, max(P, 1))
    ws = _workspace(dev, nb)
    opts = _Opts(SCHEDULES[schedule], int(lag_pairs), int(ctas_per_sm), 0, int(exp2_split),
                 int(lookahead), int(row_gap), int(engine))
    _check(_L().odpo_online_dpo_loss_fwd_bwd_ex(
        _p(policy_logits), dt, B, T, V, sb, st, _p(ref_logp), _p(tokens), _p(mask), _p(pair_rows),
        P, Pg, float(beta), float(inv_temperature), _p(dl), dl.stride(0), dl.stride(1), _p(seq),
        _p(z), _p(stats), _p(status), _p(ws), ws.numel(), C.byref(opts), _stream()),
        "odpo_online_dpo_loss_fwd_bwd")
    return LossOutput(stats, dl, seq, z[:P], status, int(opts.launches))


@_traced
def online_dpo_loss_fwd_bwd_unscaled(policy_logits: torch.Tensor, ref_logp: torch.Tensor,
                                     tokens: torch.Tensor, mask: torch.Tensor, beta: float,
                                     pair_rows: torch.Tensor | None = None,
                                     p_global: int | None = None, inv_temperature: float = 1.0,
                                     inplace: bool = False, G: torch.Tensor | None = None,
                                     row_scale: torch.Tensor | None = None, ctas_per_sm: int = 0,
                                     exp2_split: int = -1, lookahead: int = -1, row_gap: int = -1,
                                     engine: int = -1, schedule: str = "auto",
                                     stats: torch.Tensor | None = None,
                                     status: torch.Tensor | None = None) -> LossOutput:
    """The loss call with the gradient factored per row (schedule "auto" = the row engine,
    or "resident": each row's backward read back from tensor memory): out.dlogits holds
    G = mask (softmax - onehot) and out.row_scale [B, T] holds coef_b * mask, so the gradient
    is out.row_scale[..., None] * out.dlogits (one HBM read and one write of the logits)."""
    dt, B, T, V, sb, st = _logits_meta(policy_logits, "policy_logits")
    ref_logp = _per_seq(ref_logp, "ref_logp", B)
    tokens, mask = _tokmask(tokens, mask, B, T)
    dev = policy_logits.device
    pair_rows, P = _pairs(pair_rows, B)
    Pg = P if p_global is None else int(p_global)
    if inplace:
        g = policy_logits
    elif G is not None:
        g = _out_rows(G, policy_logits, "G")
    else:
        g = _rows_like(policy_logits)
    if g.dim() != 3 or g.stride(2) != 1:
        raise OdpoError("G must be [B, T, V] with a contiguous last dimension")
    if row_scale is None:
        row_scale = torch.empty((B, T), dtype=torch.float32, device=dev)
    row_scale = _dev(row_scale, "row_scale", torch.float32)
    if not row_scale.is_contiguous() or row_scale.numel() != B * T:
        raise OdpoError("row_scale must be a contiguous [B, T] f32 tensor")
    seq = torch.empty(B, dtype=torch.float32, device=dev)
    z = torch.empty(max(P, 1), dtype=torch.float32, device=dev)
    stats = _stats(stats, dev)
    status = _status(status, dev)
    ws = _workspace(dev, workspace_bytes(B, T, max(P, 1)))
    opts = _Opts(SCHEDULES[schedule], 0, int(ctas_per_sm), 0, int(exp2_split), int(lookahead),
                 int(row_gap), int(engine))
    _check(_L().odpo_online_dpo_loss_fwd_bwd_unscaled(
        _p(policy_logits), dt, B, T, V, sb, st, _p(ref_logp), _p(tokens), _p(mask), _p(pair_rows),
        P, Pg, float(beta), float(inv_temperature), _p(g), g.stride(0), g.stride(1), _p(row_scale),
        _p(seq), _p(z), _p(stats), _p(status), _p(ws), ws.numel(), C.byref(opts), _stream()),
        "odpo_online_dpo_loss_fwd_bwd_unscaled")
    return LossOutput(stats, g, seq, z[:P], status, int(opts.launches), row_scale)


PG_KINDS = {"rloo": 0, "copg": 1, "prox_rloo": 2, "sft": 3}


@_traced
def pg_loss_fwd_bwd(policy_logits: torch.Tensor, tokens: torch.Tensor, mask: torch.Tensor,
                    kind: str, rewards: torch.Tensor, old_logp: torch.Tensor | None = None,
                    clip_eps: float = 0.2, pair_rows: torch.Tensor | None = None,
                    p_global: int | None = None, inv_temperature: float = 1.0,
                    inplace: bool = False, dlogits: torch.Tensor | None = None,
                    schedule: str = "auto", ctas_per_sm: int = 0, engine: int = -1,
                    stats: torch.Tensor | None = None,
                    status: torch.Tensor | None = None) -> LossOutput:
    """App B losses on the same path: kind in rloo / copg / prox_rloo /
    sft; rewards[B] and old_logp[B] per sequence.  out.z is empty (no DPO logit)."""
    dt, B, T, V, sb, st = _logits_meta(policy_logits, "policy_logits")
    tokens, mask = _tokmask(tokens, mask, B, T)
    rewards = _per_seq(rewards, "rewards", B)
    if old_logp is not None:
        old_logp = _per_seq(old_logp, "old_logp", B)
    dev = policy_logits.device
    pair_rows, P = _pairs(pair_rows, B)
    Pg = P if p_global is None else int(p_global)
    if inplace:
        dl = policy_logits
    elif dlogits is not None:
        dl = _out_rows(dlogits, policy_logits, "dlogits")
    else:
        dl = _rows_like(policy_logits)
    if dl.dim() != 3 or dl.stride(2) != 1:
        raise OdpoError("dlogits must be [B, T, V] with a contiguous last dimension")
    seq = torch.empty(B, dtype=torch.float32, device=dev)
    stats = _stats(stats, dev)
    status = _status(status, dev)
    ws = _workspace(dev, workspace_bytes(B, T, max(P, 1)))
    opts = _Opts(SCHEDULES[schedule], 0, int(ctas_per_sm), 0, -1, -1, -1, int(engine))
    _check(_L().odpo_pg_loss_fwd_bwd(
        _p(policy_logits), dt, B, T, V, sb, st, _p(tokens), _p(mask), _p(pair_rows), P, Pg,
        PG_KINDS[kind], _p(rewards), _p(old_logp), float(clip_eps), float(inv_temperature),
        _p(dl), dl.stride(0), dl.stride(1), _p(seq), _p(stats), _p(status), _p(ws), ws.numel(),
        C.byref(opts), _stream()), "odpo_pg_loss_fwd_bwd")
    return LossOutput(stats, dl, seq, seq[:0], status, int(opts.launches))


@_traced
def vp_row_partials(logits_shard: torch.Tensor, v0: int, V_total: int, tokens: torch.Tensor,
                    mask: torch.Tensor, inv_temperature: float = 1.0,
                    status: torch.Tensor | None = None) -> torch.Tensor:
    """Vocabulary-parallel forward of one shard (columns [v0, v0 + V_shard) of V_total):
    returns the [B*T, 4] f32 row partials (m, log1p r, x_tok, owns)."""
    dt, B, T, V, sb, st = _logits_meta(logits_shard, "logits_shard")
    tokens, mask = _tokmask(tokens, mask, B, T)
    parts = torch.empty((B * T, 4), dtype=torch.float32, device=logits_shard.device)
    status = _status(status, logits_shard.device)
    ws = _workspace(logits_shard.device, workspace_bytes(B, T, B // 2 + 1))
    _check(_L().odpo_vp_row_partials(_p(logits_shard), dt, B, T, V, sb, st, int(v0), int(V_total),
                                     _p(tokens), _p(mask), float(inv_temperature), _p(parts),
                                     _p(status), _p(ws), ws.numel(), _stream()),
           "odpo_vp_row_partials")
    return parts


@_traced
def vp_loss_fwd_bwd(parts_all: torch.Tensor, logits_shard: torch.Tensor, v0: int, V_total: int,
                    ref_logp: torch.Tensor, tokens: torch.Tensor, mask: torch.Tensor, beta: float,
                    pair_rows: torch.Tensor | None = None, p_global: int | None = None,
                    inv_temperature: float = 1.0, dlogits: torch.Tensor | None = None,
                    stats: torch.Tensor | None = None, status: torch.Tensor | None = None,
                    flags: torch.Tensor | None = None, epoch: int = 0) -> LossOutput:
    """Vocabulary-parallel loss of one shard from the all-gathered partials [W, B*T, 4]:
    global log-probs, loss and stats (identical on every rank of the vocabulary group) and
    this shard's dlogits."""
    dt, B, T, V, sb, st = _logits_meta(logits_shard, "logits_shard")
    parts_all = _dev(parts_all, "parts_all", torch.float32).contiguous()
    W = parts_all.shape[0]
    if parts_all.dim() != 3 or tuple(parts_all.shape[1:]) != (B * T, 4):
        raise OdpoError(f"parts_all must be [W, B*T, 4] = [W, {B * T}, 4]")
    ref_logp = _per_seq(ref_logp, "ref_logp", B)
    tokens, mask = _tokmask(tokens, mask, B, T)
    dev = logits_shard.device
    pair_rows, P = _pairs(pair_rows, B)
    Pg = P if p_global is None else int(p_global)
    dl = _rows_like(logits_shard) if dlogits is None else _out_rows(dlogits, logits_shard, "dlogits")
    seq = torch.empty(B, dtype=torch.float32, device=dev)
    z = torch.empty(max(P, 1), dtype=torch.float32, device=dev)
    stats = _stats(stats, dev)
    status = _status(status, dev)
    ws = _workspace(dev, workspace_bytes(B, T, max(P, 1)))
    _check(_L().odpo_vp_loss_fwd_bwd(
        _p(parts_all), W, _p(logits_shard), dt, B, T, V, sb, st, int(v0), int(V_total),
        _p(ref_logp), _p(tokens), _p(mask), _p(pair_rows), P, Pg, float(beta),
        float(inv_temperature), _p(dl), dl.stride(0), dl.stride(1), _p(seq), _p(z), _p(stats),
        _p(flags), int(epoch) & 0xFFFFFFFF, _p(status), _p(ws), ws.numel(), _stream()),
        "odpo_vp_loss_fwd_bwd")
    return LossOutput(stats, dl, seq, z[:P], status, 4)


class VPExchange:
    """Peer-memory exchange buffers of the vocabulary-parallel step.

    Every rank owns one device buffer: the row partials of two epochs, [2][W][rows][4] f32
    (slot [e % 2][q] written by rank q), W u32 flag words and a u32 CTA counter, then the
    statistics slots of two epochs, [2][W][16] f64, and their W flag words (the peer-memory
    form of the stats all-reduce, `allreduce_stats(stats, exchange=...)`).  The buffers
    are mapped into every rank's address space: over the process group the ranks exchange
    CUDA IPC handles of their buffers (torch's CUDA tensor sharing) and open each other's, so
    odpo_vp_row_partials_put stores straight into the peers' memory (NVLink P2P on one node;
    IPC between processes sharing a GPU) and odpo_vp_loss_fwd_bwd waits on its own flags.
    `VPExchange.emulate(W, rows, device)` builds W ranks' buffers inside one process (tests)."""

    def __init__(self, rows: int, group=None, device=None, _bufs=None, _rank=0):
        self.rows = int(rows)
        if _bufs is not None:
            self.bufs, self.rank, self.W = _bufs, _rank, len(_bufs)
        else:
            import torch.distributed as dist
            from torch.multiprocessing.reductions import reduce_tensor
            self.W = dist.get_world_size(group)
            self.rank = dist.get_rank(group)
            if self.W > 8:
                raise OdpoError("the in-kernel exchange supports up to 8 ranks per vocabulary group")
            dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
            own = torch.zeros(self.nbytes(self.W, self.rows), dtype=torch.uint8, device=dev)
            torch.cuda.synchronize(dev)
            handles = [None] * self.W
            dist.all_gather_object(handles, reduce_tensor(own), group=group)
            self.bufs = []
            for q, (fn, args) in enumerate(handles):
                self.bufs.append(own if q == self.rank else fn(*args))
            dist.barrier(group)
        self.epoch = 0
        self.stats_epoch = 0

    @staticmethod
    def _stats_off(W: int, rows: int) -> int:
        return (2 * W * rows * 16 + 4 * W + 4 + 255) // 256 * 256

    @staticmethod
    def nbytes(W: int, rows: int) -> int:
        return VPExchange._stats_off(W, rows) + 2 * W * 128 + 4 * W + 256

    @classmethod
    def emulate(cls, W: int, rows: int, device=None):
        """W ranks' exchanges in one process (every 'peer' buffer is a local allocation)."""
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        bufs = [torch.zeros(cls.nbytes(W, rows), dtype=torch.uint8, device=dev) for _ in range(W)]
        return [cls(rows, _bufs=bufs, _rank=r) for r in range(W)]

    def _parts_ptr(self, q, e):
        return self.bufs[q].data_ptr() + (e % 2) * self.W * self.rows * 16

    def _flags_ptr(self, q):
        return self.bufs[q].data_ptr() + 2 * self.W * self.rows * 16

    def parts(self, e) -> torch.Tensor:
        """This rank's [W, rows, 4] partials of epoch e (rank q's slice written by rank q)."""
        n = self.W * self.rows * 4
        f = self.bufs[self.rank][: 2 * n * 4].view(torch.float32)
        return f[(e % 2) * n:(e % 2 + 1) * n].view(self.W, self.rows, 4)

    def flags(self) -> torch.Tensor:
        off = 2 * self.W * self.rows * 16
        return self.bufs[self.rank][off:off + 4 * self.W].view(torch.int32)

    def done(self) -> int:
        return self._flags_ptr(self.rank) + 4 * self.W

    def _sslots_ptr(self, q, e):
        return self.bufs[q].data_ptr() + self._stats_off(self.W, self.rows) + (e % 2) * self.W * 128

    def _sflags_ptr(self, q):
        return self.bufs[q].data_ptr() + self._stats_off(self.W, self.rows) + 2 * self.W * 128


@_traced
def vp_row_partials_put(logits_shard: torch.Tensor, v0: int, V_total: int, tokens: torch.Tensor,
                        mask: torch.Tensor, ex: VPExchange, epoch: int,
                        inv_temperature: float = 1.0, status: torch.Tensor | None = None):
    """Forward of this rank's shard with the exchange in the kernel: partials stored into every
    rank's buffer (peer memory) and `epoch` published to every rank's flags."""
    dt, B, T, V, sb, st = _logits_meta(logits_shard, "logits_shard")
    tokens, mask = _tokmask(tokens, mask, B, T)
    if B * T != ex.rows:
        raise OdpoError(f"exchange built for {ex.rows} rows, shard has {B * T}")
    status = _status(status, logits_shard.device)
    W = ex.W
    parts = (C.c_void_p * W)(*[ex._parts_ptr(q, epoch) for q in range(W)])
    flags = (C.c_void_p * W)(*[ex._flags_ptr(q) for q in range(W)])
    _check(_L().odpo_vp_row_partials_put(
        _p(logits_shard), dt, B, T, V, sb, st, int(v0), int(V_total), _p(tokens), _p(mask),
        float(inv_temperature), parts, flags, C.c_void_p(ex.done()), ex.rank, W,
        int(epoch) & 0xFFFFFFFF, _p(status), _stream()), "odpo_vp_row_partials_put")
    return status


@_traced
def vp_loss_step(logits_shard: torch.Tensor, v0: int, V_total: int, ref_logp: torch.Tensor,
                 tokens: torch.Tensor, mask: torch.Tensor, beta: float, group=None,
                 exchange: VPExchange | None = None, **kw) -> LossOutput:
    """One vocabulary-parallel learner step on this rank: partials, their exchange over the
    vocabulary group, loss and dlogits shard.  With `exchange` (a VPExchange) the partials move
    inside the kernels over peer memory -- two launches of ours, no host collective; without
    it they are all-gathered by the process group (NCCL over NVLink with the nccl backend)."""
    if exchange is not None:
        exchange.epoch += 1
        e = exchange.epoch
        st = vp_row_partials_put(logits_shard, v0, V_total, tokens, mask, exchange, e,
                                 kw.get("inv_temperature", 1.0), kw.get("status"))
        kw["status"] = st
        return vp_loss_fwd_bwd(exchange.parts(e), logits_shard, v0, V_total, ref_logp, tokens,
                               mask, beta, flags=exchange.flags(), epoch=e, **kw)
    import torch.distributed as dist
    parts = vp_row_partials(logits_shard, v0, V_total, tokens, mask,
                            kw.get("inv_temperature", 1.0), kw.get("status"))
    W = dist.get_world_size(group)
    if dist.get_backend(group) == "nccl":
        parts_all = torch.empty((W,) + tuple(parts.shape), dtype=parts.dtype, device=parts.device)
        dist.all_gather_into_tensor(parts_all, parts, group=group)
    else:
        chunks = [torch.empty_like(parts) for _ in range(W)]
        dist.all_gather(chunks, parts, group=group)
        parts_all = torch.stack(chunks)
    return vp_loss_fwd_bwd(parts_all, logits_shard, v0, V_total, ref_logp, tokens, mask, beta, **kw)


@_traced
def allreduce_stats(stats: torch.Tensor, group=None, exchange: "VPExchange | None" = None
                    ) -> torch.Tensor:
    """SUM all-reduce of the fp64 statistics buffer across data-parallel ranks (NCCL over
    NVLink/NVSwitch on GPU process groups; gloo for CPU tests).  One 128-byte message:
    the loss is already divided by the static P_global, so the summed buffer holds the
    global loss, accuracy numerator and margins.

    With `exchange` (a VPExchange over the same ranks) the reduction runs over peer memory
    instead (the SURVEY's K6 stretch): odpo_stats_put stores the buffer into every rank's slot
    and publishes an epoch, odpo_stats_sum waits for all W flags and sums the slots in rank
    order -- two one-warp launches of ours, no collective, the same bits on every rank."""
    if exchange is not None:
        _dev(stats, "stats", torch.float64)
        if not stats.is_contiguous() or stats.numel() < STATS_BUF:
            raise OdpoError(f"stats must be a contiguous float64 buffer of {STATS_BUF} doubles")
        exchange.stats_epoch += 1
        e = exchange.stats_epoch
        W = exchange.W
        slots = (C.c_void_p * W)(*[exchange._sslots_ptr(q, e) for q in range(W)])
        flags = (C.c_void_p * W)(*[exchange._sflags_ptr(q) for q in range(W)])
        _check(_L().odpo_stats_put(_p(stats), slots, flags, exchange.rank, W, e & 0xFFFFFFFF,
                                   _stream()), "odpo_stats_put")
        _check(_L().odpo_stats_sum(C.c_void_p(exchange._sslots_ptr(exchange.rank, e)),
                                   C.c_void_p(exchange._sflags_ptr(exchange.rank)), W,
                                   e & 0xFFFFFFFF, _p(stats), _stream()), "odpo_stats_sum")
        return stats
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=group)
    return stats


def summarize(stats: torch.Tensor) -> dict:
    """Global means from a (reduced) 16-double stats buffer."""
    s = stats.double().cpu().tolist()
    n = max(s[0], 1.0)
    return {
        "loss": s[1],
        "accuracy": s[2] / n,
        "implicit_margin": s[3] / n,
        "chosen_reward": s[4] / n,
        "rejected_reward": s[5] / n,
        "chosen_logp": s[6] / n,
        "rejected_logp": s[7] / n,
        "reward_margin": s[10] / n,
        "npairs": s[0],
        "ndegenerate": s[11],
        "ntruncated": s[12],
    }


def shard_pairs(P_global: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous pair block [p0, p1) of rank `rank`: pairs are
    independent, so each rank's logits come from its own data-parallel replica and the
    static P_global keeps dlogits identical to a single-GPU run."""
    return (rank * P_global) // world, ((rank + 1) * P_global) // world
