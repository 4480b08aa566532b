#!/usr/bin/env python
"""bench.py -- Online-DPO learner hot path on B200: pairs/s and achieved HBM GB/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config llama] [--impl ours|reference]

The default workload is BASELINE.json configs[3], LLaMA-3.1-8B No Robots (64 pairs x 2,
T 1024, V 128256, bf16): the largest configuration that fits one GPU (configs[4], the
strong-scaling sweep, is 2048 pairs of that shape; --config strong).

One STEP = one pass of the whole hot path over one batch of synthetic input
(SURVEY.md §8(a) rows S1-S6): pair_select over the rewards, the Online-DPO loss
forward + dlogits backward over the policy logits [B,T,V], and (N > 1) the SUM
all-reduce of the 128-byte statistics buffer over NCCL.  The reference log-probs
(one forward pass over a second "reference model" logits tensor) are computed once at
setup, as stored log pi_init values; that pass is timed separately ("ref_pass").

Multi-GPU: torchrun, one process per GPU; every rank processes its own contiguous
block of pairs of the same shape (weak scaling, global P = N * P_rank, static
P_global), data keyed by global pair index.  Timing: CUDA events on the launching
stream per step with an L2 flush (untimed 256 MiB write) between steps, summed,
max over ranks.  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Online DPO fwd+bwd pairs/s and achieved HBM GB/s (% of B200 peak) at 1/2/4/8 GPUs"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="llama",
                    choices=["tiny", "pythia", "rho", "llama", "strong", "rho_k4"])
    ap.add_argument("--chunk-pairs", type=int, default=64)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--schedule", default="auto", choices=["auto", "fused", "two_pass", "wave", "resident", "psync"])
    ap.add_argument("--lag", type=int, default=0)
    ap.add_argument("--ctas-per-sm", type=int, default=0)
    ap.add_argument("--exp2-split", type=int, default=-1)
    ap.add_argument("--lookahead", type=int, default=-1)
    ap.add_argument("--mask", default="dense", choices=["dense", "prefix"])
    ap.add_argument("--gradient", default="scaled", choices=["scaled", "unscaled"],
                    help="scaled: dlogits (the north_star output); unscaled: G + row_scale")
    ap.add_argument("--loss", default="dpo", choices=["dpo", "rloo", "copg", "prox_rloo", "sft"],
                    help="dpo: Online DPO (the north_star); others: App B losses on the same path")
    ap.add_argument("--row-gap", type=int, default=-1)
    ap.add_argument("--engine", type=int, default=-1, help="row-engine geometry (-1 auto)")
    ap.add_argument("--no-aux", action="store_true",
                    help="skip the auxiliary timing of the other gradient form")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--stats-exchange", action="store_true",
                    help="N > 1: the statistics SUM over peer memory (odpo_stats_put/_sum through "
                         "a VPExchange: CUDA IPC / NVLink P2P) instead of the NCCL all-reduce")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="issue every timed step from Python instead of replaying CUDA graphs of "
                         "the step's library calls (the replays keep the GPU fed: no host "
                         "marshalling gap inside the timed region)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--lib", default=None,
                    help="A/B experiments only: load this build of libodpo.so instead of the "
                         "in-tree one (e.g. build_variants/*.so from build.build(out=, defines=))")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, b.copy_ read+write)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def bf16_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        if "bf16_tflops" in d:
            return float(d["bf16_tflops"]), "measured (MEASURED_PEAKS.json bf16_tflops, cuBLAS)"
    return 1590.0, "fallback (B200_PROFILING.md)"


def src_sha() -> str:
    """Hash of the sources the loss call's kernels are compiled from (odpo.cu and the headers
    it includes, the C header; not odpo_lmhead.cu, whose NEXT-2 kernels the captured loss
    call never launches): an ncu capture is used as this run's traffic evidence only if it was
    taken on the same sources."""
    import glob
    import hashlib
    h = hashlib.sha256()
    files = sorted(f for f in glob.glob(os.path.join(ROOT, "paper_2410_18252_b200", "csrc", "*.cu*"))
                   if not f.endswith("odpo_lmhead.cu"))
    for f in files + [os.path.join(ROOT, "include", "odpo.h")]:
        h.update(open(f, "rb").read())
    return h.hexdigest()[:16]


def ncu_evidence(config, form):
    """ncu --set full record of this config's dominant kernel (profiles/r02/ncu/), or None when
    there is none for the current sources."""
    p = os.path.join(ROOT, "profiles", "r02", "ncu", f"traffic_{config}_{form}.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    if d.get("src_sha") != src_sha():
        return None
    d["file"] = os.path.relpath(p, ROOT)
    return d


def measure_ceilings(dev):
    """Copy and read-only HBM ceilings measured in this run: b.copy_(a) over
    1 Gi bf16 (read + write bytes, MEASURED_PEAKS.json's method) and a read-only 128-bit stream
    over 4 GiB (read bytes), best of 5 with CUDA events."""
    import torch
    out = {}
    a = torch.empty(1 << 30, dtype=torch.bfloat16, device=dev)
    b = torch.empty_like(a)
    a.fill_(1.0)

    def best(fn, nbytes):
        fn()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return nbytes / (min(ts) / 1e3) / 1e9

    out["copy_gbs"] = best(lambda: b.copy_(a), 2 * a.numel() * 2)
    del a, b
    x = torch.empty(2 << 30, dtype=torch.bfloat16, device=dev)
    x.fill_(0.5)
    import synth
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    out["read_gbs"] = max(best(lambda: synth.read_probe(x, sms * k), x.numel() * 2) for k in (8, 16))
    del x
    torch.cuda.empty_cache()
    out["how"] = ("copy: b.copy_(a) 1 Gi bf16, read+write bytes; read: a 128-bit read-only stream "
                  "over 4 GiB (synth_read_probe, 8 loads in flight per thread); best of 5")
    return out


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# LM-head shapes of the paper's models (hidden width d, vocabulary V) for the NEXT-2 aux line
HEADS = {"pythia": (2560, 50304), "rho": (2048, 32000)}


def aux_lmhead(config, B, T, reps=5):
    """NEXT-2 forward (odpo_lmhead_seq_logprobs: tcgen05 GEMM + online log-softmax, logits never
    stored) on the config's model head, beside cuBLAS's bf16 GEMM + odpo_seq_logprobs."""
    import torch

    import paper_2410_18252_b200 as odpo
    if config not in HEADS:
        return None
    d, V = HEADS[config]
    g = torch.Generator(device="cuda").manual_seed(0)
    hid = (torch.randint(-32, 32, (B, T, d), device="cuda", generator=g).float() / 32).to(torch.bfloat16)
    Wh = (torch.randint(-32, 32, (V, d), device="cuda", generator=g).float() / 256).to(torch.bfloat16)
    tok = torch.randint(0, V, (B, T), device="cuda", generator=g, dtype=torch.int32)
    msk = torch.ones((B, T), dtype=torch.uint8, device="cuda")

    def t(fn):
        for _ in range(2):
            fn()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(reps)]
        torch.cuda.synchronize()
        for a, b in ev:
            a.record()
            fn()
            b.record()
        torch.cuda.synchronize()
        return float(np.median([a.elapsed_time(b) for a, b in ev]))

    fused = t(lambda: odpo.lmhead_seq_logprobs(hid, Wh, tok, msk))
    gemm = t(lambda: torch.matmul(hid.view(B * T, d), Wh.t()))
    lg = torch.matmul(hid.view(B * T, d), Wh.t()).view(B, T, V)
    seqp = t(lambda: odpo.seq_logprobs(lg, tok, msk))
    del lg
    # the full head learner step: fused (logits never stored; backward recomputes them in
    # wave-sized row chunks, tcgen05 GEMMs for dhidden / dweight) vs unfused (cuBLAS logits, the
    # loss call in place, two cuBLAS GEMMs)
    ref_h = torch.full((B,), -4.0 * T, device="cuda")

    def fused_step():
        o = odpo.lmhead_online_dpo_loss_fwd(hid, Wh, ref_h, tok, msk, 0.1)
        return odpo.lmhead_grad(hid, Wh, tok, o.row_lse, o.row_scale)

    def unfused_step():
        lg2 = torch.matmul(hid.view(B * T, d), Wh.t()).view(B, T, V)
        o = odpo.online_dpo_loss_fwd_bwd(lg2, ref_h, tok, msk, 0.1, inplace=True)
        dl = o.dlogits.view(B * T, V)
        return torch.matmul(dl, Wh), torch.matmul(dl.t(), hid.view(B * T, d))

    def chunked_step():
        return odpo.lmhead_dpo_step(hid, Wh, ref_h, tok, msk, 0.1)

    step_c = t(chunked_step)
    o_h = odpo.lmhead_online_dpo_loss_fwd(hid, Wh, ref_h, tok, msk, 0.1)
    grad_ms = t(lambda: odpo.lmhead_grad(hid, Wh, tok, o_h.row_lse, o_h.row_scale))
    step_f = t(fused_step)
    step_u = t(unfused_step)
    del hid, Wh
    torch.cuda.empty_cache()
    flops = 2.0 * B * T * d * V
    pk, src = bf16_peak()
    return {"kernel": "odpo_lmhead_seq_logprobs (k_lmhead_fwd2 + merge)", "rows": B * T, "d": d,
            "V": V, "bound": "tensor", "ms": fused, "achieved": flops / fused / 1e9,
            "unit": "TFLOP/s", "peak": pk, "peak_source": src, "frac": flops / fused / 1e9 / pk,
            "cublas_gemm_ms": gemm, "cublas_tflops": flops / gemm / 1e9,
            "unfused_ms": gemm + seqp, "speedup_vs_unfused": (gemm + seqp) / fused,
            "step_fused_ms": step_f, "step_unfused_ms": step_u, "step_chunked_ms": step_c,
            "step_chunked_note": "odpo_lmhead_dpo_step: per ~1 GB chunk of whole pairs, bf16 "
                                 "logits (own tcgen05 GEMM), the loss call in place, dhidden / "
                                 "dweight (own tcgen05 GEMMs): three head GEMMs, one chunk of "
                                 "logits in memory",
            "grad_ms": grad_ms, "grad_tflops": 3 * flops / grad_ms / 1e9,
            "grad_note": "odpo_lmhead_grad alone: logits recompute + G epilogue, dhidden and "
                         "dweight GEMMs (3 x 2 R d V flops) on the library's tcgen05 kernels",
            "step_note": "fwd + DPO loss + dhidden/dweight; fused keeps no logits (backward "
                         "recomputes them in wave-sized row chunks and runs its own tcgen05 "
                         "GEMMs), unfused materialises them (cuBLAS GEMMs)"}


class ClockSampler:
    """NVML SM-clock / throttle-reason sampler running during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.stop_ev = [], 0, threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self.stop_ev.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        names = [n for bit, n in self.REASONS.items() if self.reasons & bit and bit != 0x1]
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples)}


def workload(name):
    from synth.configs import CONFIGS
    return CONFIGS[name]


# ----------------------------------------------------------------------------- oracle timing
_SAMPLES: dict = {}


def oracle_inputs(w, seed, npairs, mask_kind, p0=0):
    """Host inputs of npairs pairs of the workload (synth, untimed; cached)."""
    key = (w.name, seed, npairs, mask_kind, p0)
    if key in _SAMPLES:
        return _SAMPLES[key]
    import oracle
    import synth
    K = w.K
    seqs = np.arange(K * npairs) + K * p0
    rows = (seqs[:, None] * w.T + np.arange(w.T)[None, :]).reshape(-1)
    tok_all = synth.tokens_rows(seed, rows, w.V).reshape(-1, w.T)
    mask_all = synth.mask_for(seed, seqs, w.T, mask_kind, w.lbar)
    rewards = synth.rewards_for(seed, npairs, K, p0=p0, kind=w.reward_kind)
    eos = synth.has_eos_for(seed, npairs, K, p0=p0) if w.eos_penalty is not None else None
    pen = w.eos_penalty if w.eos_penalty is not None else 0.0
    # K > 2: logits exist for the selected pair only
    sel_rows = oracle.pair_select(rewards, eos, pen)["pair_rows"].reshape(-1) if K > 2 \
        else np.arange(2 * npairs)
    tok, mask = tok_all[sel_rows], mask_all[sel_rows]
    grow = (seqs[sel_rows][:, None] * w.T + np.arange(w.T)[None, :]).reshape(-1)
    x = synth.logits_rows(seed, grow, w.V, tokens=tok.reshape(-1), peak=14.0).astype(np.float32)
    x = x.reshape(len(sel_rows), w.T, w.V)
    if w.dtype == "bf16":
        x = oracle.to_bf16_bits(x)
    ref = np.full(len(sel_rows), -0.08 * w.T, np.float32)
    _SAMPLES.clear()
    _SAMPLES[key] = (x, tok, mask, rewards, eos, pen, ref)
    return _SAMPLES[key]


def oracle_sample(w, seed, npairs, mask_kind, n_threads, p0=0):
    """Time the CPU oracle (as it stands) on npairs pairs of the same workload: pair_select,
    the fp64 loss and the full dlogits."""
    import oracle
    x, tok, mask, rewards, eos, pen, ref = oracle_inputs(w, seed, npairs, mask_kind, p0)
    t0 = time.perf_counter()
    sel = oracle.pair_select(rewards, eos, pen)
    o = oracle.online_dpo_loss_fwd_bwd(x, ref, tok, mask, w.beta,
                                       pair_rows=sel["pair_rows"] if w.K == 2 else None,
                                       want_dlogits=True, n_threads=n_threads)
    dt = time.perf_counter() - t0
    return dt, o


def oracle_pairs_per_sample(w, cores):
    """A bounded sample: whole pairs, about 2e7 logits per sample at most (one LLaMA pair is
    2.6e8 and is the unit there)."""
    per_pair = 2 * w.T * w.V
    return int(max(1, min(w.P, cores, 2e7 // per_pair)))


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle is this tier's reference arm (rank 0 only)."""
    if rank != 0:
        return
    w = workload(args.config)
    cores = os.cpu_count() or 1
    npairs = oracle_pairs_per_sample(w, cores)
    threads = cores
    for _ in range(max(0, min(args.warmup, 1))):
        oracle_sample(w, args.seed, npairs, args.mask, threads)
    times = []
    for _ in range(args.steps):
        dt, _ = oracle_sample(w, args.seed, npairs, args.mask, threads)
        times.append(dt)
    tot = float(np.sum(times))
    value = npairs * len(times) / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "pairs/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "pairs_per_step": npairs, "T": w.T, "V": w.V,
                   "logits_dtype": w.dtype, "mask": args.mask},
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": threads, "kind": "oracle",
                         "cpu_model": cpu_model(),
                         "sample": f"{npairs} pairs of {args.config} per step (pair_select + "
                                   f"loss + full dlogits, fp64, {threads} threads)"},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- ours
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import synth
    import paper_2410_18252_b200 as odpo
    if args.lib:
        odpo.LIB_PATH = os.path.abspath(args.lib)

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    ceil = measure_ceilings(dev)
    w = workload(args.config)
    P, T, V = w.P, w.T, w.V
    B = 2 * P
    p0 = rank * P                       # global pair offset of this rank
    Pg = P * world
    tdt = torch.bfloat16 if w.dtype == "bf16" else torch.float32
    s_in = 2 if w.dtype == "bf16" else 4
    Kc = w.K                            # completions per prompt
    n_src = Kc * P                      # completions of this rank
    if Kc > 2 and args.loss != "dpo":
        raise SystemExit("App B losses are benchmarked with K = 2 configs")
    seqs = np.arange(n_src) + Kc * p0
    rows = (seqs[:, None] * T + np.arange(T)[None, :]).reshape(-1)

    # ---------------- inputs (untimed): rewards, tokens, mask on device; logits via device twin
    rewards = torch.from_numpy(synth.rewards_for(args.seed, P, Kc, p0=p0, kind=w.reward_kind)).to(dev)
    eos = (torch.from_numpy(synth.has_eos_for(args.seed, P, Kc, p0=p0)).to(dev)
           if w.eos_penalty is not None else None)
    pen = w.eos_penalty if w.eos_penalty is not None else 0.0
    tokens_all = torch.from_numpy(synth.tokens_rows(args.seed, rows, V).reshape(n_src, T)).to(dev)
    mask_all = torch.from_numpy(synth.mask_for(args.seed, seqs, T, args.mask, w.lbar)).to(dev)
    if Kc > 2:
        # K completions per prompt, only the selected pair is trained on: the
        # policy logits exist for the 2P selected completions, compacted by odpo_gather_pairs
        sel0 = odpo.pair_select(rewards, eos, pen)
        tokens, mask, _ = odpo.gather_pairs(sel0.pair_rows, tokens_all, mask_all)
    else:
        sel0 = None
        tokens, mask = tokens_all, mask_all
    torch.cuda.synchronize()
    rho = float(mask.float().mean().item())
    logits = torch.empty((B, T, V), dtype=tdt, device=dev)
    dlogits = torch.empty_like(logits)

    # reference model log-probs: one forward pass over independent "reference" logits
    synth.fill_logits_device(logits, args.seed, row0=int(rows[0]), tokens=tokens, peak=14.0, ref=True)
    torch.cuda.synchronize()
    ref_logp = odpo.seq_logprobs(logits, tokens, mask)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ref_ms = []
    for _ in range(3):
        e0.record()
        ref_logp = odpo.seq_logprobs(logits, tokens, mask)
        e1.record()
        torch.cuda.synchronize()
        ref_ms.append(e0.elapsed_time(e1))
    synth.fill_logits_device(logits, args.seed, row0=int(rows[0]), tokens=tokens, peak=14.0)
    # per-completion offsets in [-32, 32) nats on the stored reference log-probs (hash stream
    # 14, keyed by the global completion index): the synthetic reference model is the policy's
    # twin, so without them z ~ 0 and the loss ~ ln 2; with them z spreads across the sigmoid
    # (saturating for |z| >~ 1) as with a real reference model.  Inputs only: no cost change.
    if Kc == 2:
        off = synth.hash_u64(args.seed, 14, (np.arange(B) + 2 * p0))
        ref_logp = ref_logp + torch.from_numpy(((off % np.uint64(256)).astype(np.float64) - 128.0)
                                               / 4.0).to(dev).float()
    if Kc > 2:
        # per-completion reference log-probs (the selected ones from the pass above)
        ref_all = torch.full((n_src,), -0.08 * T, dtype=torch.float32, device=dev)
        off = synth.hash_u64(args.seed, 14, seqs)
        ref_all[sel0.pair_rows.reshape(-1).long()] = ref_logp
        ref_all = ref_all + torch.from_numpy(((off % np.uint64(256)).astype(np.float64) - 128.0)
                                             / 4.0).to(dev).float()
    else:
        ref_all = ref_logp
    torch.cuda.synchronize()

    stats = torch.zeros(16, dtype=torch.float64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    row_scale = torch.empty((B, T), dtype=torch.float32, device=dev)
    sx = odpo.VPExchange(1) if (args.stats_exchange and world > 1) else None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    launches = [0]

    rew_seq = rewards.reshape(-1).contiguous()   # per-sequence rewards (App B losses)

    def loss_call(gradient, pair_rows, ref, tok, msk):
        if args.loss != "dpo":
            # ref doubles as log pi_old for CoPG / Proximal RLOO
            return odpo.pg_loss_fwd_bwd(logits, tok, msk, args.loss, rew_seq, ref, 0.2,
                                        pair_rows=pair_rows, p_global=Pg, dlogits=dlogits,
                                        schedule=args.schedule, ctas_per_sm=args.ctas_per_sm,
                                        engine=args.engine, stats=stats, status=status)
        if gradient == "unscaled":
            return odpo.online_dpo_loss_fwd_bwd_unscaled(
                logits, ref, tok, msk, w.beta, pair_rows=pair_rows, p_global=Pg, G=dlogits,
                row_scale=row_scale, ctas_per_sm=args.ctas_per_sm, exp2_split=args.exp2_split,
                lookahead=args.lookahead, row_gap=args.row_gap, engine=args.engine, stats=stats,
                status=status, schedule="resident" if args.schedule == "resident" else "auto")
        return odpo.online_dpo_loss_fwd_bwd(logits, ref, tok, msk, w.beta, pair_rows=pair_rows,
                                            p_global=Pg, dlogits=dlogits, schedule=args.schedule,
                                            lag_pairs=args.lag, ctas_per_sm=args.ctas_per_sm,
                                            exp2_split=args.exp2_split, lookahead=args.lookahead,
                                            engine=args.engine, row_gap=args.row_gap, stats=stats,
                                            status=status)

    def step(timed_loss=None, gradient=args.gradient):
        sel = odpo.pair_select(rewards, eos, pen, status=status, sel_stats=stats[10:13])
        if Kc > 2:
            tok_g, msk_g, ref_g = odpo.gather_pairs(sel.pair_rows, tokens_all, mask_all, ref_all,
                                                    status=status)
            if timed_loss is not None:
                timed_loss[0].record()
            out = loss_call(gradient, None, ref_g, tok_g, msk_g)
            if timed_loss is not None:
                timed_loss[1].record()
            odpo.allreduce_stats(stats, exchange=sx)
            launches[0] = 2 + out.launches
            return out
        if timed_loss is not None:
            timed_loss[0].record()
        out = loss_call(gradient, sel.pair_rows, ref_logp, tokens, mask)
        if timed_loss is not None:
            timed_loss[1].record()
        odpo.allreduce_stats(stats, exchange=sx)
        launches[0] = 1 + out.launches
        return out

    def graphed(gradient):
        """The step as two CUDA graphs sharing one memory pool -- (A) pair_select (+ gather for
        K > 2), (B) the loss call -- replayed A then B; the statistics all-reduce stays eager
        between replays (a collective).  Each replay launches exactly the library's kernels of
        one eager step, on the same buffers; only the Python marshalling leaves the timed
        region.  Returns a step(timed_loss) closure, or None when capture fails (eager)."""
        if args.no_graph or args.stats_exchange:
            return None
        try:
            pool = torch.cuda.graph_pool_handle()
            gA, gB = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):     # the capture stream's workspace, allocated eagerly
                sel_w = odpo.pair_select(rewards, eos, pen, status=status, sel_stats=stats[10:13])
                loss_call(gradient, sel_w.pair_rows if Kc == 2 else None, ref_logp, tokens, mask)
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            keep = {}
            with torch.cuda.graph(gA, pool=pool, stream=side):
                sel = odpo.pair_select(rewards, eos, pen, status=status, sel_stats=stats[10:13])
                keep["sel"] = sel
                if Kc > 2:
                    keep["g"] = odpo.gather_pairs(sel.pair_rows, tokens_all, mask_all, ref_all,
                                                  status=status)
            with torch.cuda.graph(gB, pool=pool, stream=side):
                if Kc > 2:
                    tok_g, msk_g, ref_g = keep["g"]
                    keep["out"] = loss_call(gradient, None, ref_g, tok_g, msk_g)
                else:
                    keep["out"] = loss_call(gradient, sel.pair_rows, ref_logp, tokens, mask)
            torch.cuda.synchronize()
        except Exception as e:   # noqa: BLE001 -- report and time the eager step instead
            print(f"bench: CUDA graph capture failed ({e}); timing eager steps", file=sys.stderr)
            torch.cuda.synchronize()
            return None

        def gstep(timed_loss=None, gradient=gradient):
            gA.replay()
            if timed_loss is not None:
                timed_loss[0].record()
            gB.replay()
            if timed_loss is not None:
                timed_loss[1].record()
            odpo.allreduce_stats(stats, exchange=sx)
            return keep["out"]
        gstep.keep = keep
        return gstep

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    gstep_main = graphed(args.gradient)
    if gstep_main is not None:
        for _ in range(2):
            gstep_main()
        torch.cuda.synchronize()
    timed_step = gstep_main if gstep_main is not None else step
    if world > 1:
        dist.barrier()

    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    lev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    clk = ClockSampler(local_rank)
    with clk:
        for k in range(K):
            flush.zero_()                      # untimed L2 flush between steps
            torch.cuda.synchronize()
            ev[k][0].record()
            timed_step(lev[k])
            ev[k][1].record()
        torch.cuda.synchronize()
    step_ms = np.array([a.elapsed_time(b) for a, b in ev])
    loss_ms = np.array([a.elapsed_time(b) for a, b in lev])
    n_launch = launches[0]
    tot = torch.tensor([step_ms.sum()], dtype=torch.float64, device=dev)
    if world > 1:
        dist.barrier()
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    tot_ms = float(tot.item())
    value = world * P * K / (tot_ms / 1e3)
    st = int(status.item())
    # the replayed graphs compute what an eager step computes: same statistics, same dlogits
    graph_check = None
    if gstep_main is not None and world == 1:
        g_stats, g_dl = stats[:10].clone(), dlogits.view(-1)[:: 4099].clone()
        step()
        torch.cuda.synchronize()
        graph_check = bool(torch.equal(g_stats, stats[:10]) and torch.equal(g_dl, dlogits.view(-1)[:: 4099]))

    # algorithmic bytes per loss launch: read the live rows once, write every dlogit once
    alg_bytes = rho * B * T * V * s_in + B * T * V * s_in
    achieved = alg_bytes / (loss_ms.mean() / 1e3) / 1e9
    peak, peak_src = peaks()

    # the other gradient form on the same inputs, timed the same way and reported beside the
    # headline (scaled dlogits = the north_star output; factored = G + row_scale)
    form = ("scaled" if args.gradient == "scaled" else "unscaled") if args.loss == "dpo" else args.loss
    aux = None
    if not args.no_aux and args.loss == "dpo":
        other = "unscaled" if args.gradient == "scaled" else "scaled"
        for _ in range(2):
            step(gradient=other)
        torch.cuda.synchronize()
        gstep_aux = graphed(other)
        aux_step = gstep_aux if gstep_aux is not None else (lambda t: step(t, gradient=other))
        aux_step(None)
        aev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(K)]
        for k in range(K):
            flush.zero_()
            torch.cuda.synchronize()
            aux_step(aev[k])
        torch.cuda.synchronize()
        ams = np.array([a.elapsed_time(b) for a, b in aev])
        aach = alg_bytes / (ams.mean() / 1e3) / 1e9
        nv = ncu_evidence(args.config, other)
        aux = {"gradient": other, "bound": "hbm", "achieved": aach, "peak": peak, "unit": "GB/s",
               "frac": aach / peak, "frac_of_copy_ceiling": aach / ceil["copy_gbs"],
               "traffic": nv["dram_bytes_per_launch"] if nv else None,
               "ncu": nv, "loss_ms_mean": float(ams.mean()),
               "pairs_per_s_loss_only": world * P / (ams.mean() / 1e3),
               "alg_bytes_per_launch": alg_bytes, "status": int(status.item()),
               "kernel": ("odpo_online_dpo_loss_fwd_bwd_unscaled (prep + fwd/bwd)" if other == "unscaled"
                          else "odpo_online_dpo_loss_fwd_bwd (AUTO = two-pass)")}
    # NEXT-2 aux: the Pythia-2.8B LM head (the head whose fused step VERDICT r1 asks to beat)
    lmh = aux_lmhead("pythia", 512, 53) if not args.no_aux and args.loss == "dpo" else None
    nv_main = ncu_evidence(args.config, form)
    traffic = nv_main["dram_bytes_per_launch"] if nv_main else None
    # 2R+1W: the scaled output's traffic floor where a pair does not fit in L2
    floor_bytes = 2 * rho * B * T * V * s_in + B * T * V * s_in

    # ---------------- e2e through host buffers (pinned H2D inputs, D2H stats + z each step)
    e2e = None
    if not args.no_e2e:
        # every rank pins one step's inputs (33.6 GB for LLaMA): check the host can hold all the
        # node's ranks' buffers, and agree across ranks, before any of them starts the e2e loop
        need = logits.numel() * s_in
        ok, reason = 1, ""
        try:
            import psutil
            nloc = int(os.environ.get("LOCAL_WORLD_SIZE", world))
            avail = psutil.virtual_memory().available
            if avail < 1.25 * need * nloc:
                ok, reason = 0, (f"host memory: {avail / 1e9:.0f} GB available for {nloc} pinned "
                                 f"buffers of {need / 1e9:.1f} GB")
        except ImportError:
            pass
        h_logits = None
        if ok:
            try:
                h_logits = torch.empty(logits.shape, dtype=tdt, pin_memory=True)
            except RuntimeError as e:
                ok, reason = 0, f"pinned host allocation failed: {e}"[:200]
        if world > 1:
            t_ok = torch.tensor([ok], dtype=torch.int32, device=dev)
            dist.all_reduce(t_ok, op=dist.ReduceOp.MIN)
            if int(t_ok.item()) == 0 and ok:
                ok, reason = 0, "another rank could not pin its host buffer"
        if not ok:
            e2e = {"unavailable": reason}
            h_logits = None
        else:
            h_logits.copy_(logits)
            h_rew = rewards.cpu().pin_memory()
            h_eos = eos.cpu().pin_memory() if eos is not None else None
            h_tok = tokens_all.cpu().pin_memory()
            h_mask = mask_all.cpu().pin_memory()
            h_ref = ref_all.cpu().pin_memory()
            h_stats = torch.empty(16, dtype=torch.float64, pin_memory=True)
            h_z = torch.empty(P, dtype=torch.float32, pin_memory=True)
            d_rew, d_tok, d_mask, d_ref = (torch.empty_like(rewards), torch.empty_like(tokens_all),
                                           torch.empty_like(mask_all), torch.empty_like(ref_all))
            d_eos = torch.empty_like(eos) if eos is not None else None
            h2d = (h_logits.numel() * s_in + h_rew.numel() * 4 + (h_eos.numel() if h_eos is not None else 0)
                   + h_tok.numel() * 4 + h_mask.numel() + h_ref.numel() * 4)
            d2h = 16 * 8 + P * 4

            def e2e_step():
                logits.copy_(h_logits, non_blocking=True)
                d_rew.copy_(h_rew, non_blocking=True)
                if d_eos is not None:
                    d_eos.copy_(h_eos, non_blocking=True)
                d_tok.copy_(h_tok, non_blocking=True)
                d_mask.copy_(h_mask, non_blocking=True)
                d_ref.copy_(h_ref, non_blocking=True)
                sel = odpo.pair_select(d_rew, d_eos, pen, status=status, sel_stats=stats[10:13])
                if Kc > 2:
                    tg, mg, rg = odpo.gather_pairs(sel.pair_rows, d_tok, d_mask, d_ref, status=status)
                    out = loss_call(args.gradient, None, rg, tg, mg)
                else:
                    out = loss_call(args.gradient, sel.pair_rows, d_ref, d_tok, d_mask)
                odpo.allreduce_stats(stats, exchange=sx)
                h_stats.copy_(stats, non_blocking=True)
                h_z.copy_(out.z, non_blocking=True)

            e2e_step()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(args.e2e_steps):
                e2e_step()
            b.record()
            torch.cuda.synchronize()
            et = torch.tensor([a.elapsed_time(b)], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(et, op=dist.ReduceOp.MAX)
            e2e = {"value": world * P * args.e2e_steps / (float(et.item()) / 1e3), "unit": "pairs/s",
                   "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                   "steps": args.e2e_steps,
                   "note": "pinned host->device copy of logits, rewards, eos, tokens, mask, ref_logp; "
                           "device->host of the stats buffer and per-pair z; dlogits stay resident "
                           "for the LM-head backward"}
            del h_logits

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        # the oracle as it stands, on one block of this workload's pairs repeated until about
        # args.cpu_seconds of CPU work have been timed (a bounded sample), on every host core;
        # then the same block once on ONE core
        del dlogits, logits
        torch.cuda.empty_cache()
        cores = os.cpu_count() or 1
        npairs = oracle_pairs_per_sample(w, cores)
        done, spent = 0, 0.0
        while spent < args.cpu_seconds and done < 64 * P:
            dt, _ = oracle_sample(w, args.seed, npairs, args.mask, cores)
            spent += dt
            done += npairs
        dt1, _ = oracle_sample(w, args.seed, npairs, args.mask, 1)
        cpu = {"value": done / spent, "unit": "pairs/s", "cores": cores, "kind": "oracle",
               "cpu_model": cpu_model(),
               "sample": f"{done} pairs of the {args.config} workload in blocks of {npairs} "
                         f"(pair_select + fp64 loss + full dlogits), {spent:.1f} s on {cores} "
                         f"host threads",
               "single_thread": {"value": npairs / dt1, "unit": "pairs/s", "cores": 1,
                                 "sample": f"{npairs} pairs, {dt1:.1f} s on one thread"}}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": tot_ms / K, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": w.dtype, "data": "synthetic",
            "config": {"workload": args.config, "pairs_per_rank": P, "global_pairs": P * world,
                       "K": Kc, "T": T, "V": V, "beta": w.beta, "mask": args.mask,
                       "ref_logp": "seq_logprobs over independent reference logits (setup) + "
                                   "per-completion offsets in [-32, 32) nats (z spread)",
                       "schedule": args.schedule, "exp2_split": args.exp2_split,
                       "loss": args.loss, "gradient": args.gradient, "engine": args.engine,
                       "parallelism": f"dp{world}",
                       "launch": ("CUDA graph replays of the step's library calls (pair_select; "
                                  "the loss call), statistics reduction eager"
                                  if gstep_main is not None else "eager Python calls"),
                       "graph_matches_eager": graph_check,
                       "stats_reduction": ("peer memory (odpo_stats_put/_sum)" if args.stats_exchange
                                           and world > 1 else "NCCL all_reduce" if world > 1 else "none"),
                       "l2": "inputs (%.2f GB) > L2; plus 256 MiB L2 flush between timed steps"
                             % (B * T * V * s_in / 1e9)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "frac_of_copy_ceiling": achieved / ceil["copy_gbs"],
                         "frac_of_8tbs_spec": achieved / 8000.0,
                         "ncu_dram_gbs": (traffic / (loss_ms.mean() / 1e3) / 1e9) if traffic else None,
                         "floor_bytes_per_launch": floor_bytes if form == "scaled" else None,
                         "floor_frac": (floor_bytes / (loss_ms.mean() / 1e3) / 1e9 / peak
                                        if form == "scaled" else None),
                         "floor_note": ("2R+1W: the backward of a pair re-reads its rows, which "
                                        "do not stay in L2 between the pair's forward pass and "
                                        "its coefficient (DESIGN.md 4)" if form == "scaled" else None),
                         "ncu": nv_main,
                         "kernel": ("odpo_pg_loss_fwd_bwd (%s)" % args.loss if args.loss != "dpo"
                                    else "odpo_online_dpo_loss_fwd_bwd (AUTO = two-pass: prep, "
                                         "forward, pair reduction, backward)"
                                    if args.gradient == "scaled" else
                                    "odpo_online_dpo_loss_fwd_bwd_unscaled (prep + fwd/bwd)"),
                         "alg_bytes_per_launch": alg_bytes,
                         "loss_ms_mean": float(loss_ms.mean())},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(n_launch * K),
            "roofline_factored" if form == "scaled" else "roofline_other_form": aux,
            "ceilings": ceil,
            "aux_lmhead_pythia": lmh,
            "clocks": clk.summary(),
            "tokens_vocab_per_s": world * B * T * V * K / (tot_ms / 1e3),
            "eff_gbs_step": world * alg_bytes * K / (tot_ms / 1e3) / 1e9,
            "step_ms_p10_p50_p90": [float(np.percentile(step_ms, q)) for q in (10, 50, 90)],
            "ref_pass_ms": float(np.median(ref_ms)),
            "ref_pass_gbs": rho * B * T * V * s_in / (np.median(ref_ms) / 1e3) / 1e9,
            "status": st,
            "loss": float(stats[1].item()),
        }
        print(json.dumps(line), flush=True)



# ----------------------------------------------------------------------------- strong scaling
def run_strong(args, rank, world, local_rank):
    """BASELINE.json configs[4]: 2048 pairs, T=1024, V=128256, bf16, batch-sharded over the
    ranks (strong scaling: total work fixed).  Each rank owns a contiguous block of pairs and
    processes it in LLaMA-shaped chunks of --chunk-pairs pairs with in-place dlogits (the
    1.08 TB of logits never fit at once); chunk logits are regenerated on the device OUTSIDE
    the timed region.  Per step the timed region is, per chunk, pair_select + the fused
    loss fwd+bwd, plus one stats all-reduce; chunk times are summed; max over ranks."""
    import torch
    import torch.distributed as dist

    import synth
    import paper_2410_18252_b200 as odpo

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    w = workload("strong")
    T, V, Pg = w.T, w.V, w.P
    p_lo, p_hi = odpo.shard_pairs(Pg, world, rank)
    C = args.chunk_pairs
    chunks = [(p, min(p + C, p_hi)) for p in range(p_lo, p_hi, C)]
    logits = torch.empty((2 * C, T, V), dtype=torch.bfloat16, device=dev)
    stats = torch.zeros(16, dtype=torch.float64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    acc = torch.zeros(16, dtype=torch.float64, device=dev)
    sx = odpo.VPExchange(1) if (args.stats_exchange and world > 1) else None
    ref_val = -0.1 * T

    def prep_chunk(c0, c1):
        n = c1 - c0
        seqs = np.arange(2 * c0, 2 * c1)
        rows = (seqs[:, None] * T + np.arange(T)[None, :]).reshape(-1)
        tok = torch.from_numpy(synth.tokens_rows(args.seed, rows, V).reshape(2 * n, T)).to(dev)
        mask = torch.from_numpy(synth.mask_for(args.seed, seqs, T, args.mask, w.lbar)).to(dev)
        rew = torch.from_numpy(synth.rewards_for(args.seed, n, 2, p0=c0)).to(dev)
        eos = torch.from_numpy(synth.has_eos_for(args.seed, n, 2, p0=c0)).to(dev)
        x = logits[:2 * n]
        synth.fill_logits_device(x, args.seed, row0=int(rows[0]), tokens=tok, peak=14.0)
        ref = torch.full((2 * n,), ref_val, dtype=torch.float32, device=dev)
        return x, tok, mask, rew, eos, ref, float(mask.float().mean().item())

    meta = {}

    def one_step(timed):
        total_ms, loss_ms, alg = 0.0, 0.0, 0.0
        acc.zero_()
        for (c0, c1) in chunks:
            x, tok, mask, rew, eos, ref, rho = prep_chunk(c0, c1)
            torch.cuda.synchronize()
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record()
            sel = odpo.pair_select(rew, eos, w.eos_penalty, status=status, sel_stats=stats[10:13])
            e[1].record()
            out = odpo.online_dpo_loss_fwd_bwd(x, ref, tok, mask, w.beta, pair_rows=sel.pair_rows,
                                               p_global=Pg, inplace=True, schedule=args.schedule,
                                               lag_pairs=args.lag, exp2_split=args.exp2_split,
                                               stats=stats, status=status)
            acc.add_(stats)
            e[2].record()
            torch.cuda.synchronize()
            total_ms += e[0].elapsed_time(e[2])
            loss_ms += e[1].elapsed_time(e[2])
            alg += (rho + 1.0) * x.numel() * 2
            meta["launches"] = 1 + out.launches
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        odpo.allreduce_stats(acc, exchange=sx)
        e1.record()
        torch.cuda.synchronize()
        total_ms += e0.elapsed_time(e1)
        return total_ms, loss_ms, alg

    for _ in range(args.warmup):
        one_step(False)
    if world > 1:
        dist.barrier()
    clk = ClockSampler(local_rank)
    tot, ltot, alg = 0.0, 0.0, 0.0
    with clk:
        for _ in range(args.steps):
            a, b_, c = one_step(True)
            tot += a
            ltot += b_
            alg += c
    t = torch.tensor([tot], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tmax = float(t.item())
    peak, peak_src = peaks()
    achieved = alg / (ltot / 1e3) / 1e9
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": Pg * args.steps / (tmax / 1e3), "unit": "pairs/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": tmax / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": "strong", "global_pairs": Pg, "T": T, "V": V,
                       "chunk_pairs": C, "pairs_rank0": p_hi - p_lo, "mask": args.mask,
                       "parallelism": f"dp{world}", "inplace": True,
                       "l2": "each chunk (33.6 GB) > L2; logits regenerated between chunks"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None, "peak_source": peak_src,
                         "kernel": "odpo_online_dpo_loss_fwd_bwd (rank 0 chunks)"},
            "cpu_baseline": None, "e2e": None,
            "gpu_launches": int(meta.get("launches", 0) * len(chunks) * args.steps),
            "clocks": clk.summary(),
            "tokens_vocab_per_s": 2 * Pg * T * V * args.steps / (tmax / 1e3),
            "loss": float(acc[1].item()),
        }), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        # ODPO_DIST_BACKEND=gloo + ODPO_SHARE_GPU=1: several ranks on one GPU (tests the
        # multi-rank path on a 1-GPU box; NCCL refuses duplicate devices)
        if os.environ.get("ODPO_SHARE_GPU") == "1":
            local_rank = local_rank % max(1, torch.cuda.device_count())
        torch.cuda.set_device(local_rank)
        backend = os.environ.get("ODPO_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    try:
        if args.config == "strong":
            run_strong(args, rank, world, local_rank)
        else:
            run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
