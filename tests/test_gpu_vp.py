"""NEXT-4: vocabulary-parallel loss, W shards of the vocabulary emulated on one GPU (the
all-gather of the row partials is a torch.stack here; NCCL all_gather_into_tensor across
ranks in vp_loss_step).  Compared with the unsharded oracle."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_helpers import NCPU, Batch, check_dlogits, check_seq, check_stats, coef_from_oracle, to_f64

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def odpo():
    import paper_2410_18252_b200 as m
    m._L()
    return m


def shard_bounds(V, W, align):
    """W contiguous column ranges, inner boundaries on multiples of `align` elements (the
    16-byte alignment of every shard base)."""
    cuts = [0] + [((V * w) // W) // align * align for w in range(1, W)] + [V]
    return list(zip(cuts[:-1], cuts[1:]))


@pytest.mark.parametrize("W", [1, 3, 8, 40])
@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_vp_parity(odpo, W, dt):
    """W = 40 > 32 partials per row take the warp-per-row merge (k_vp_combine_wide)."""
    P, T, V = 3, 9, 12345 if dt == "f32" else 32000
    b = Batch(P, T, V, dt, seed=7, mask_kind="prefix", lbar=5, extra_seqs=1)
    ref = (synth.rewards_for(7, b.B, 1).reshape(-1) - 20.0).astype(np.float32)
    d_ref = torch.from_numpy(ref).cuda()
    align = 8 if dt == "bf16" else 4
    bounds = shard_bounds(V, W, align)
    parts = [odpo.vp_row_partials(b.d_logits[:, :, a:e], a, V, b.d_tokens, b.d_mask)
             for a, e in bounds]
    parts_all = torch.stack(parts)
    dl = b.new_out()
    outs = [odpo.vp_loss_fwd_bwd(parts_all, b.d_logits[:, :, a:e], a, V, d_ref, b.d_tokens,
                                 b.d_mask, 0.1, pair_rows=b.d_pair_rows, p_global=P + 1,
                                 dlogits=dl[:, :, a:e]) for a, e in bounds]
    torch.cuda.synchronize()
    o = oracle.online_dpo_loss_fwd_bwd(b.h_logits, ref, b.tokens, b.mask, 0.1,
                                       pair_rows=b.pair_rows, p_global=P + 1, want_dlogits=True,
                                       n_threads=NCPU)
    live = b.pair_rows.reshape(-1)
    for out in outs:   # every rank of the vocabulary group holds the same global results
        assert torch.equal(out.seq_logp[torch.from_numpy(live).cuda()],
                           outs[0].seq_logp[torch.from_numpy(live).cuda()])
        assert torch.equal(out.stats[:10], outs[0].stats[:10])
        assert int(out.status.item()) == 0
    check_seq(outs[0].seq_logp.cpu().numpy()[live], o["seq_logp"][live], dt)
    check_stats(outs[0].stats.cpu().numpy(), o, dt, 0.1, ref, b.pair_rows, Pg=P + 1)
    coef = coef_from_oracle(o, P, P + 1, 0.1, 1.0, b.pair_rows, b.B)
    check_dlogits(to_f64(dl), o["dlogits"], coef[:, None, None], dt)


def test_vp_token_ownership_flags(odpo):
    """A token outside [0, V_total) is flagged; every in-range token has exactly one owner."""
    b = Batch(2, 5, 4096, "bf16", seed=8, host=False)
    parts = [odpo.vp_row_partials(b.d_logits[:, :, a:e], a, 4096, b.d_tokens, b.d_mask)
             for a, e in shard_bounds(4096, 4, 8)]
    owners = torch.stack(parts)[:, :, 3].sum(0)
    assert torch.all(owners[b.d_mask.reshape(-1).bool()] == 1)
    tok = b.d_tokens.clone()
    tok[0, 0] = 4096
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    odpo.vp_row_partials(b.d_logits[:, :, 0:2048], 0, 4096, tok, b.d_mask, status=st)
    torch.cuda.synchronize()
    assert int(st.item()) & odpo.FLAGS["TOKEN_RANGE"]


# ------------------------------------------------------------------ in-kernel exchange
def _vp_case(W, dt, seed=9):
    P, T, V = 3, 9, 32000 if dt == "bf16" else 12345
    b = Batch(P, T, V, dt, seed=seed, mask_kind="prefix", lbar=5, extra_seqs=1)
    ref = (synth.rewards_for(seed, b.B, 1).reshape(-1) - 20.0).astype(np.float32)
    align = 8 if dt == "bf16" else 4
    return b, torch.from_numpy(ref).cuda(), shard_bounds(V, W, align)


@pytest.mark.parametrize("W", [2, 3, 8])
@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_vp_in_kernel_exchange_matches_gather(odpo, W, dt):
    """The partials exchanged INSIDE the kernels (odpo_vp_row_partials_put stores into every
    rank's buffer and publishes the epoch; the merge waits on its flags) give the same bits as
    the gathered path, for two consecutive epochs (both halves of the double buffer)."""
    b, d_ref, bounds = _vp_case(W, dt)
    P, rows = b.P, b.B * b.T
    ex = odpo.VPExchange.emulate(W, rows)
    for epoch in (1, 2, 3):
        parts = torch.stack([odpo.vp_row_partials(b.d_logits[:, :, a:e], a, b.V, b.d_tokens, b.d_mask)
                             for a, e in bounds])
        for r, (a, e) in enumerate(bounds):   # every rank's put (one stream: all land first)
            st = odpo.vp_row_partials_put(b.d_logits[:, :, a:e], a, b.V, b.d_tokens, b.d_mask,
                                          ex[r], epoch)
            assert int(st.item()) == 0
        for r, (a, e) in enumerate(bounds):
            assert torch.equal(ex[r].parts(epoch), parts)
            assert ex[r].flags().tolist() == [epoch] * W
            dl_g, dl_x = b.new_out(), b.new_out()
            g = odpo.vp_loss_fwd_bwd(parts, b.d_logits[:, :, a:e], a, b.V, d_ref, b.d_tokens,
                                     b.d_mask, 0.1, pair_rows=b.d_pair_rows, p_global=P + 1,
                                     dlogits=dl_g[:, :, a:e])
            x = odpo.vp_loss_fwd_bwd(ex[r].parts(epoch), b.d_logits[:, :, a:e], a, b.V, d_ref,
                                     b.d_tokens, b.d_mask, 0.1, pair_rows=b.d_pair_rows,
                                     p_global=P + 1, dlogits=dl_x[:, :, a:e],
                                     flags=ex[r].flags(), epoch=epoch)
            torch.cuda.synchronize()
            assert torch.equal(g.stats[:10], x.stats[:10]) and torch.equal(g.z, x.z)
            assert torch.equal(dl_g[:, :, a:e], dl_x[:, :, a:e])
        for r in range(W):   # every rank's CTA counter is back at 0 after its put kernel
            off = 2 * W * rows * 16 + 4 * W
            assert int(ex[r].bufs[r][off:off + 4].view(torch.int32).item()) == 0


def _vp_proc(rank, world, port, q):
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2410_18252_b200 as odpo
        torch.cuda.set_device(0)
        b, d_ref, bounds = _vp_case(world, "bf16", seed=12)
        a, e = bounds[rank]
        ex = odpo.VPExchange(b.B * b.T)
        res = []
        for _ in range(3):
            out = odpo.vp_loss_step(b.d_logits[:, :, a:e].contiguous(), a, b.V, d_ref, b.d_tokens,
                                    b.d_mask, 0.1, exchange=ex, pair_rows=b.d_pair_rows,
                                    p_global=b.P + 1)
            torch.cuda.synchronize()
            res.append((out.stats[:10].cpu().numpy(), out.dlogits.float().cpu().numpy(),
                        int(out.status.item())))
        # the unsharded loss on the full logits (the same process computes it for comparison)
        full = odpo.online_dpo_loss_fwd_bwd(b.d_logits, d_ref, b.d_tokens, b.d_mask, 0.1,
                                            pair_rows=b.d_pair_rows, p_global=b.P + 1)
        torch.cuda.synchronize()
        # the statistics all-reduce over peer memory between the two processes
        st = torch.arange(16, dtype=torch.float64, device="cuda") * (rank + 1) + 0.125
        odpo.allreduce_stats(st, exchange=ex)
        torch.cuda.synchronize()
        # plain numpy (pickled): no shared-memory handles that die with this process
        q.put((rank, res, full.stats[:10].cpu().numpy(),
               full.dlogits[:, :, a:e].float().cpu().numpy(), st.cpu().numpy()))
    finally:
        dist.destroy_process_group()


def test_vp_exchange_two_processes(odpo):
    """World size 2 with real process boundaries: two ranks (processes) on this GPU exchange the
    partials through each other's memory (CUDA IPC handles swapped over a gloo group), three
    steps in a row; every step equals the unsharded loss (stats within fp32 rounding of the
    merge, dlogits within one bf16 ulp) and the two ranks agree exactly on the global stats."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_vp_proc, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(2):
        r, res, fs, fdl, st = q.get(timeout=300)
        got[r] = ([(torch.from_numpy(a), torch.from_numpy(b), c) for a, b, c in res],
                  torch.from_numpy(fs), torch.from_numpy(fdl))
        exp = (np.arange(16) * 1.0 + 0.125) + (np.arange(16) * 2.0 + 0.125)
        assert np.array_equal(st, exp)   # peer-memory stats all-reduce: the rank-order sum
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in (0, 1):
        res, fs, fdl = got[r]
        for st, dl, status in res:
            assert status == 0
            assert torch.equal(st, res[0][0]) and torch.equal(dl, res[0][1])  # step-to-step
            assert st[0] == fs[0] and st[8] == fs[8] and st[9] == fs[9]
            assert torch.allclose(st, fs, rtol=1e-5, atol=1e-9)
            assert torch.all((dl - fdl).abs() <= 2.0 ** -7 * fdl.abs() + 1e-12)
    assert torch.equal(got[0][0][0][0], got[1][0][0][0])


@pytest.mark.parametrize("W", [2, 3, 8])
def test_stats_allreduce_over_peer_memory(odpo, W):
    """The statistics SUM over peer memory (odpo_stats_put / odpo_stats_sum): every emulated
    rank gets exactly the rank-order sum, for two epochs (both halves of the double buffer)."""
    import ctypes as C
    ex = odpo.VPExchange.emulate(W, 1)
    L = odpo._L()
    rng = np.random.default_rng(W)
    for epoch in (1, 2, 3):
        loc = [torch.from_numpy(rng.normal(size=16)).cuda() for _ in range(W)]
        for r in range(W):
            slots = (C.c_void_p * W)(*[ex[r]._sslots_ptr(q, epoch) for q in range(W)])
            flags = (C.c_void_p * W)(*[ex[r]._sflags_ptr(q) for q in range(W)])
            assert L.odpo_stats_put(C.c_void_p(loc[r].data_ptr()), slots, flags, r, W, epoch,
                                    None) == 0
        outs = [torch.empty(16, dtype=torch.float64, device="cuda") for _ in range(W)]
        for r in range(W):
            assert L.odpo_stats_sum(C.c_void_p(ex[r]._sslots_ptr(r, epoch)),
                                    C.c_void_p(ex[r]._sflags_ptr(r)), W, epoch,
                                    C.c_void_p(outs[r].data_ptr()), None) == 0
        torch.cuda.synchronize()
        exp = np.zeros(16)
        for q in range(W):
            exp = exp + loc[q].cpu().numpy()
        for r in range(W):
            assert np.array_equal(outs[r].cpu().numpy(), exp)
