"""Multi-process (world size 2, gloo, CPU) coverage of the N>1 host logic: contiguous pair
shards with a static P_global plus ONE SUM all-reduce of the 16-double statistics buffer
reproduce the unsharded statistics (the oracle computes each shard; the product's
allreduce_stats does the exchange)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import synth
    import paper_2410_18252_b200 as odpo
    P, T, V, seed, beta = 10, 4, 37, 3, 0.1
    p0, p1 = odpo.shard_pairs(P, world, rank)
    seqs = np.arange(2 * p0, 2 * p1)
    rows = (seqs[:, None] * T + np.arange(T)[None, :]).reshape(-1)
    tok = synth.tokens_rows(seed, rows, V).reshape(-1, T)
    x = synth.logits_rows(seed, rows, V, tokens=tok.reshape(-1)).reshape(-1, T, V).astype(np.float32)
    mask = synth.mask_for(seed, seqs, T, "prefix", 2)
    rewards = synth.rewards_for(seed, p1 - p0, 2, p0=p0)
    sel = oracle.pair_select(rewards, None, -1.0)
    ref = np.full(len(seqs), -3.0, np.float32)
    o = oracle.online_dpo_loss_fwd_bwd(x, ref, tok, mask, beta, pair_rows=sel["pair_rows"], p_global=P)
    buf = torch.zeros(16, dtype=torch.float64)
    buf[:10] = torch.from_numpy(o["stats"])
    buf[10:13] = torch.from_numpy(sel["sel_stats"])
    odpo.allreduce_stats(buf)
    torch.save(buf, os.path.join(out_dir, f"r{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_stats_allreduce_gloo(tmp_path, world):
    import oracle
    import synth
    port = _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    bufs = [torch.load(tmp_path / f"r{r}.pt") for r in range(world)]
    for b in bufs[1:]:
        assert torch.equal(b, bufs[0])           # every rank holds the same global stats
    P, T, V, seed, beta = 10, 4, 37, 3, 0.1
    seqs = np.arange(2 * P)
    rows = (seqs[:, None] * T + np.arange(T)[None, :]).reshape(-1)
    tok = synth.tokens_rows(seed, rows, V).reshape(-1, T)
    x = synth.logits_rows(seed, rows, V, tokens=tok.reshape(-1)).reshape(-1, T, V).astype(np.float32)
    mask = synth.mask_for(seed, seqs, T, "prefix", 2)
    sel = oracle.pair_select(synth.rewards_for(seed, P, 2), None, -1.0)
    ref = np.full(2 * P, -3.0, np.float32)
    o = oracle.online_dpo_loss_fwd_bwd(x, ref, tok, mask, beta, pair_rows=sel["pair_rows"])
    g = bufs[0].numpy()
    assert np.allclose(g[:10], o["stats"], rtol=1e-12, atol=1e-12)
    for i in (0, 2, 8, 9):
        assert g[i] == o["stats"][i]
    assert np.allclose(g[10:13], sel["sel_stats"], rtol=1e-12, atol=0)
    assert np.all(g[13:] == 0)


def test_shard_pairs_partition():
    import paper_2410_18252_b200 as odpo
    for P in (1, 7, 64, 2048):
        for W in (1, 2, 4, 8):
            spans = [odpo.shard_pairs(P, W, r) for r in range(W)]
            assert spans[0][0] == 0 and spans[-1][1] == P
            assert all(spans[i][1] == spans[i + 1][0] for i in range(W - 1))
