"""C-ABI boundary checks that need no GPU: libodpo.so loads, exports every symbol that
include/odpo.h declares, and rejects bad arguments synchronously (before any launch)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "odpo.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2410_18252_b200 import build
    build.build()
    import paper_2410_18252_b200 as odpo
    return odpo._L()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(odpo_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_three_paper_calls():
    fns = declared_functions()
    for f in ("odpo_pair_select", "odpo_seq_logprobs", "odpo_online_dpo_loss_fwd_bwd",
              "odpo_workspace_bytes", "odpo_status_string"):
        assert f in fns


def test_library_exports_every_declared_symbol(lib):
    so = os.path.join(ROOT, "paper_2410_18252_b200", "libodpo.so")
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (odpo_\w+)", out))
    for f in declared_functions():
        assert f in exported, f
        assert hasattr(lib, f)


def test_header_compiles_as_c():
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-fsyntax-only", "-x", "c", HEADER],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_status_strings_and_version(lib):
    for code in range(6):
        assert lib.odpo_status_string(code)
    assert b"sm_100a" in lib.odpo_version()


def test_workspace_bytes(lib):
    n = lib.odpo_workspace_bytes(512, 53, 256)
    rows = 512 * 53
    assert 12 * rows <= n <= 12 * rows + 512 * 20 + 256 * 100 + 16 * 256
    assert lib.odpo_workspace_bytes(0, 5, 1) == 0


FAKE = C.c_void_p(0x7000_0000_0000)  # never dereferenced: validation returns first
FAKE_MIS = C.c_void_p(0x7000_0000_0008)


def _loss(lib, **kw):
    a = dict(logits=FAKE, dt=1, B=4, T=3, V=64, sb=192, st=64, ref=FAKE, tok=FAKE, mask=FAKE,
             pr=None, P=2, Pg=2, beta=0.1, invT=1.0, dl=FAKE, dsb=192, dst=64, seq=FAKE, z=None,
             stats=FAKE, status=None, ws=FAKE, wsb=1 << 20)
    a.update(kw)
    return lib.odpo_online_dpo_loss_fwd_bwd(a["logits"], a["dt"], a["B"], a["T"], a["V"], a["sb"],
                                            a["st"], a["ref"], a["tok"], a["mask"], a["pr"], a["P"],
                                            a["Pg"], a["beta"], a["invT"], a["dl"], a["dsb"],
                                            a["dst"], a["seq"], a["z"], a["stats"], a["status"],
                                            a["ws"], a["wsb"], None)


def test_argument_errors_are_synchronous(lib):
    assert _loss(lib, beta=0.0) == 1
    assert _loss(lib, beta=float("nan")) == 1
    assert _loss(lib, invT=-1.0) == 1
    assert _loss(lib, Pg=1) == 1
    assert _loss(lib, P=3) == 1            # pair_rows NULL requires B == 2P
    assert _loss(lib, st=63, sb=189) == 1  # stride_t < V
    assert _loss(lib, logits=None) == 1
    assert _loss(lib, dl=None) == 1
    assert _loss(lib, dt=7) == 1
    assert _loss(lib, logits=FAKE_MIS) == 2
    assert _loss(lib, st=68, sb=204) == 2  # 136-byte bf16 row stride: not 16-byte aligned
    assert _loss(lib, dl=FAKE_MIS) == 2
    assert _loss(lib, wsb=16) == 3
    assert _loss(lib, ws=None) == 3
    assert _loss(lib, dl=FAKE, dsb=96, dst=32) == 1   # dlogits rows overlap
    # in place requires identical strides
    assert _loss(lib, dl=FAKE, logits=FAKE, dsb=256, dst=64) == 1
    assert lib.odpo_pair_select(FAKE, None, -1.0, 4, 1, FAKE, FAKE, None, None, None, None, None) == 1
    assert lib.odpo_pair_select(None, None, -1.0, 4, 2, FAKE, FAKE, None, None, None, None, None) == 1
    assert lib.odpo_seq_logprobs(FAKE, 1, 4, 3, 64, 192, 64, FAKE, FAKE, 0.0, FAKE, None, None,
                                 None, FAKE, 1 << 20, None) == 1
    assert lib.odpo_seq_logprobs(FAKE, 1, 4, 3, 64, 192, 64, FAKE, FAKE, 1.0, FAKE, None, None,
                                 None, FAKE, 8, None) == 3


def _unscaled(lib, row_scale=FAKE, sched=0, **kw):
    a = dict(logits=FAKE, dt=1, B=4, T=3, V=64, sb=192, st=64, ref=FAKE, tok=FAKE, mask=FAKE,
             pr=None, P=2, Pg=2, beta=0.1, invT=1.0, dl=FAKE, dsb=192, dst=64, seq=FAKE, z=None,
             stats=FAKE, status=None, ws=FAKE, wsb=1 << 20)
    a.update(kw)
    import paper_2410_18252_b200 as odpo
    opts = odpo._Opts(sched, 0, 0, 0, -1, -1, -1, -1)
    return lib.odpo_online_dpo_loss_fwd_bwd_unscaled(
        a["logits"], a["dt"], a["B"], a["T"], a["V"], a["sb"], a["st"], a["ref"], a["tok"],
        a["mask"], a["pr"], a["P"], a["Pg"], a["beta"], a["invT"], a["dl"], a["dsb"], a["dst"],
        row_scale, a["seq"], a["z"], a["stats"], a["status"], a["ws"], a["wsb"], C.byref(opts),
        None)


def test_unscaled_argument_errors_are_synchronous(lib):
    assert _unscaled(lib, row_scale=None) == 1
    assert _unscaled(lib, beta=0.0) == 1
    assert _unscaled(lib, dl=None) == 1
    assert _unscaled(lib, dl=FAKE_MIS) == 2
    assert _unscaled(lib, wsb=16) == 3
    assert _unscaled(lib, sched=2) == 4    # only the AUTO schedule exists for this call
    assert _unscaled(lib, dl=FAKE, logits=FAKE, dsb=256, dst=64) == 1


def test_pg_and_gather_argument_errors_are_synchronous(lib):
    import paper_2410_18252_b200 as odpo

    def pg(kind=0, rewards=FAKE, old=None, eps=0.2, sched=0, dl=FAKE):
        opts = odpo._Opts(sched, 0, 0, 0, -1, -1, -1, -1)
        return lib.odpo_pg_loss_fwd_bwd(FAKE, 1, 4, 3, 64, 192, 64, FAKE, FAKE, None, 2, 2, kind,
                                        rewards, old, eps, 1.0, dl, 192, 64, FAKE, FAKE, None,
                                        FAKE, 1 << 20, C.byref(opts), None)
    assert pg(kind=7) == 1
    assert pg(rewards=None) == 1
    assert pg(kind=1, old=None) == 1          # CoPG needs log pi_old
    assert pg(kind=2, old=FAKE, eps=1.5) == 1  # clip range
    assert pg(dl=FAKE_MIS) == 2
    assert pg(sched=9) == 4
    assert lib.odpo_gather_pairs(None, 2, 8, 5, FAKE, FAKE, None, FAKE, FAKE, None, None, None) == 1
    assert lib.odpo_gather_pairs(FAKE, 2, 8, 0, FAKE, FAKE, None, FAKE, FAKE, None, None, None) == 1
    assert lib.odpo_gather_pairs(FAKE, 2, 8, 5, None, FAKE, None, FAKE, FAKE, None, None, None) == 1
    assert lib.odpo_gather_pairs(FAKE, 0, 8, 5, None, None, None, None, None, None, None, None) == 0


def test_product_has_no_oracle_or_cpu_fallback():
    """The product package never imports the oracle and refuses CPU tensors."""
    pkg = os.path.join(ROOT, "paper_2410_18252_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "liboracle" not in text, f
                assert "orc_" not in text, f
    import torch
    import paper_2410_18252_b200 as odpo
    with pytest.raises(odpo.OdpoError):
        odpo.pair_select(torch.zeros(3, 2))


def test_lmhead_and_token_logp_argument_errors(lib):
    """NEXT-2 calls: argument errors are synchronous return codes, no GPU needed."""
    import paper_2410_18252_b200 as odpo
    L = odpo._L()
    ws = odpo._L().odpo_lmhead_workspace_bytes(2, 3, 1000)
    assert ws > 0 and L.odpo_lmhead_workspace_bytes(0, 3, 1000) == 0

    def head(**kw):
        a = dict(h=FAKE, w=FAKE, B=2, T=3, d=128, V=1000, tok=FAKE, mask=FAKE, invT=1.0,
                 tlp=None, lse=None, seq=FAKE, status=None, ws=FAKE, wsb=ws)
        a.update(kw)
        return L.odpo_lmhead_seq_logprobs(a["h"], a["w"], a["B"], a["T"], a["d"], a["V"],
                                          a["tok"], a["mask"], a["invT"], a["tlp"], a["lse"],
                                          a["seq"], a["status"], a["ws"], a["wsb"], None)
    assert head(h=None) == 1 and head(seq=None) == 1 and head(B=0) == 1 and head(invT=0.0) == 1
    assert head(d=100) == 4                       # d % 64 != 0
    assert head(h=FAKE_MIS) == 2                  # 16-byte alignment
    assert head(wsb=16) == 3 and head(ws=None) == 3

    def tl(**kw):
        a = dict(tlp=FAKE, B=4, T=3, ref=FAKE, mask=FAKE, pr=None, P=2, Pg=2, beta=0.1, invT=1.0,
                 seq=FAKE, z=None, stats=FAKE, rs=None, status=None, ws=FAKE, wsb=1 << 20)
        a.update(kw)
        return L.odpo_online_dpo_loss_from_token_logp(
            a["tlp"], a["B"], a["T"], a["ref"], a["mask"], a["pr"], a["P"], a["Pg"], a["beta"],
            a["invT"], a["seq"], a["z"], a["stats"], a["rs"], a["status"], a["ws"], a["wsb"], None)
    assert tl(tlp=None) == 1 and tl(stats=None) == 1 and tl(P=0) == 1 and tl(Pg=1) == 1
    assert tl(beta=-1.0) == 1 and tl(B=5) == 1    # B != 2P without pair_rows
    assert tl(wsb=16) == 3


def test_lmhead_grad_argument_errors(lib):
    import paper_2410_18252_b200 as odpo
    L = odpo._L()
    sb = L.odpo_lmhead_grad_scratch_bytes(256, 128, 1000)
    # one chunk of G (bf16) + 256 bytes of slack + 256 for the CTA-pair kernels' tile counter
    assert sb >= 256 * 1000 * 2 + 256 and sb <= 256 * 1000 * 2 + 512
    assert L.odpo_lmhead_grad_scratch_bytes(0, 128, 10) == 0

    def grad(**kw):
        a = dict(h=FAKE, w=FAKE, R=100, d=128, V=1000, tok=FAKE, lse=FAKE, rs=FAKE, invT=1.0,
                 dh=FAKE, dw=FAKE, sc=FAKE, scb=sb, chunk=256)
        a.update(kw)
        return L.odpo_lmhead_grad(a["h"], a["w"], a["R"], a["d"], a["V"], a["tok"], a["lse"],
                                  a["rs"], a["invT"], a["dh"], a["dw"], a["sc"], a["scb"],
                                  a["chunk"], None)
    assert grad(h=None) == 1 and grad(rs=None) == 1 and grad(R=0) == 1 and grad(chunk=0) == 1
    assert grad(invT=float("nan")) == 1 and grad(d=96) == 4 and grad(w=FAKE_MIS) == 2
    assert grad(scb=16) == 3 and grad(sc=None) == 3


def test_seq_ppl_argument_errors(lib):
    """odpo_seq_ppl (KL proxy): outputs required, then seq_logprobs' checks."""
    def call(ppl=FAKE, ps=FAKE, invT=1.0, wsb=1 << 20, logits=FAKE):
        return lib.odpo_seq_ppl(logits, 1, 4, 3, 64, 192, 64, FAKE, FAKE, invT, FAKE, ppl, ps,
                                None, FAKE, wsb, None)
    assert call(ppl=None) == 1
    assert call(ps=None) == 1
    assert call(invT=0.0) == 1
    assert call(logits=FAKE_MIS) == 2
    assert call(wsb=8) == 3


def test_library_has_no_environment_lookups():
    """Tuning knobs are build-time defines: the product sources never read the environment
    (the statically linked CUDA runtime does, for its own CUDA_* variables)."""
    csrc = os.path.join(ROOT, "paper_2410_18252_b200", "csrc")
    for f in os.listdir(csrc):
        src = open(os.path.join(csrc, f)).read()
        assert "getenv" not in src, f
    binding = open(os.path.join(ROOT, "paper_2410_18252_b200", "__init__.py")).read()
    assert "os.environ" not in binding


def test_vp_put_argument_errors(lib):
    """odpo_vp_row_partials_put: peer arrays required, 1 <= W <= 8, 0 <= rank < W."""
    P = C.c_void_p

    def call(W=2, rank=0, parts=True, flags=True, done=FAKE, mis=False):
        pp = (P * 8)(*([FAKE_MIS if mis else FAKE] * 8)) if parts else None
        ff = (P * 8)(*([FAKE] * 8)) if flags else None
        return lib.odpo_vp_row_partials_put(FAKE, 1, 4, 3, 64, 192, 64, 0, 64, FAKE, FAKE, 1.0,
                                            pp, ff, done, rank, W, 1, None, None)
    import paper_2410_18252_b200  # noqa: F401  (argtypes registered by _L)
    assert call(parts=False) == 1 and call(flags=False) == 1 and call(done=None) == 1
    assert call(W=0) == 1 and call(W=9) == 1 and call(rank=2) == 1 and call(rank=-1) == 1
    assert call(mis=True) == 2


def test_vp_exchange_layout():
    """VPExchange buffer layout (host arithmetic, no GPU): two epochs of [W][rows][4] f32
    partials, then W flag words, then the CTA counter, all inside the buffer and disjoint."""
    import torch
    import paper_2410_18252_b200 as odpo
    W, rows = 3, 10
    bufs = [torch.zeros(odpo.VPExchange.nbytes(W, rows), dtype=torch.uint8) for _ in range(W)]
    ex = odpo.VPExchange(rows, _bufs=bufs, _rank=1)
    base = bufs[1].data_ptr()
    assert ex._parts_ptr(1, 0) == base and ex._parts_ptr(1, 1) == base + W * rows * 16
    assert ex._parts_ptr(1, 2) == ex._parts_ptr(1, 0)
    assert ex._flags_ptr(1) == base + 2 * W * rows * 16
    assert ex.done() == ex._flags_ptr(1) + 4 * W
    assert ex.done() + 4 <= base + bufs[1].numel()
    assert ex.parts(1).shape == (W, rows, 4) and ex.parts(1).data_ptr() == ex._parts_ptr(1, 1)
    assert ex.flags().numel() == W and ex.flags().data_ptr() == ex._flags_ptr(1)
    assert ex._parts_ptr(2, 1) == bufs[2].data_ptr() + W * rows * 16


def test_stats_exchange_argument_errors(lib):
    """odpo_stats_put / odpo_stats_sum (the stats SUM over peer memory): pointers and 1 <= W <= 8."""
    P = C.c_void_p
    arr = (P * 8)(*([FAKE] * 8))
    import paper_2410_18252_b200  # noqa: F401
    assert lib.odpo_stats_put(None, arr, arr, 0, 2, 1, None) == 1
    assert lib.odpo_stats_put(FAKE, None, arr, 0, 2, 1, None) == 1
    assert lib.odpo_stats_put(FAKE, arr, arr, 2, 2, 1, None) == 1
    assert lib.odpo_stats_put(FAKE, arr, arr, 0, 9, 1, None) == 1
    assert lib.odpo_stats_sum(None, FAKE, 2, 1, FAKE, None) == 1
    assert lib.odpo_stats_sum(FAKE, FAKE, 0, 1, FAKE, None) == 1
    assert lib.odpo_stats_sum(FAKE, FAKE, 2, 1, None, None) == 1


def test_tracing_toggle_wraps_public_calls():
    """NVTX tracing: every public call is wrapped, the flag is off by default."""
    import paper_2410_18252_b200 as odpo
    assert odpo._TRACE is False
    for n in ("pair_select", "seq_logprobs", "online_dpo_loss_fwd_bwd", "lmhead_dpo_step",
              "vp_loss_step", "allreduce_stats"):
        assert getattr(odpo, n).__wrapped__.__name__ == n
    odpo.set_tracing(True)
    assert odpo._TRACE is True
    odpo.set_tracing(False)
