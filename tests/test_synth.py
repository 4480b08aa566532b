"""The seeded generator: deterministic, keyed by global index, values exact in bf16/fp32,
and its host key schedule equals the CUDA twin's (host-callable symbol, no GPU)."""
import numpy as np

import synth


def test_deterministic_and_global_keys():
    a = synth.logits_rows(0, np.arange(10, 14), 777, tokens=np.arange(4), peak=14.0)
    b = synth.logits_rows(0, np.arange(0, 14), 777, tokens=np.r_[np.zeros(10, int), np.arange(4)],
                          peak=14.0)[10:]
    assert np.array_equal(a, b)
    assert not np.array_equal(a, synth.logits_rows(1, np.arange(10, 14), 777))


def test_values_on_grid_and_bf16_exact():
    x = synth.logits_rows(3, np.arange(5), 4096, peak=None)
    assert np.all(x * 64 == np.round(x * 64)) and x.min() >= -2 and x.max() < 2
    f = x.astype(np.float32)
    bits = f.view(np.uint32)
    assert np.all(bits & 0xFFFF == 0)  # representable in bf16


def test_tokens_masks_rewards():
    t = synth.tokens_rows(0, np.arange(1000), 50304)
    assert t.min() >= 0 and t.max() < 50304
    m = synth.mask_for(0, np.arange(200), 1024, "prefix", 290)
    L = m.sum(1)
    assert L.min() >= 1 and L.max() <= 579 and 200 < L.mean() < 380
    r = synth.rewards_for(0, 256, 2)
    assert r.dtype == np.float32 and np.all(r * 256 == np.round(r * 256))
    v = synth.rewards_for(0, 256, 4, kind="verifier")
    assert set(np.unique(v).tolist()) <= {0.0, 1.0}
    e = synth.has_eos_for(0, 4096, 2)
    assert 0.9 < e.mean() < 0.995


def test_device_twin_key_schedule():
    synth.build_device()
    L = synth._dev_lib()
    for seed in (0, 1, 12345):
        for stream in (1, 2, 3):
            assert L.synth_stream_key(seed, stream) == int(synth.stream_key(seed, stream))
