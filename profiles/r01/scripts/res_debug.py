"""RESIDENT schedule timeline (debug build, -DODPO_RES_DEBUG): per pair-row ticket the global
timer at claim, forward merged, coefficient acquired, backward done.  Prints the per-stage
latencies and the throughput over time.  Usage (on the GPU box):
  ODPO_LIB=build_variants/libodpo_resdbg.so python profiles/res_debug.py [P T V]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2410_18252_b200 as odpo  # noqa: E402
from gpu_helpers import Batch  # noqa: E402

P, T, V = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (256, 53, 50304)
b = Batch(P, T, V, "bf16", seed=0, host=False)
ref = torch.full((b.B,), -float(T) * 0.08, device="cuda")
out = b.new_out()
for i in range(4):
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    o = odpo.online_dpo_loss_fwd_bwd(b.d_logits, ref, b.d_tokens, b.d_mask, 0.1, schedule="resident",
                                     dlogits=out)
    t1.record()
    torch.cuda.synchronize()
    print("call ms", t0.elapsed_time(t1), "status", int(o.status.item()))
n = P * 2 * T
buf = np.zeros((n, 8), np.uint64)
rc = odpo._L().odpo_res_debug_dump(buf.ctypes.data_as(C.c_void_p), C.c_int64(n))
assert rc == 0, rc
t = (buf[:, :7].astype(np.float64) - float(buf[:, 0].min())) / 1e3  # us
print("span us", t.max())
d = np.diff(t, axis=1)
for k, name in enumerate(["claim->first chunk", "first->last chunk", "last chunk->merged",
                          "merged->coef", "coef->bwd start", "bwd start->done"]):
    print(f"{name:22s} mean {d[:, k].mean():7.2f} p10 {np.percentile(d[:, k], 10):7.2f} "
          f"p50 {np.percentile(d[:, k], 50):7.2f} p90 {np.percentile(d[:, k], 90):7.2f} us")
life = t[:, 6] - t[:, 0]
print("lifetime mean", life.mean(), "p90", np.percentile(life, 90))
# pair completion: last forward of the pair minus first claim of the pair
tp = t.reshape(P, 2 * T, 7)
print("pair claim span mean", (tp[:, :, 0].max(1) - tp[:, :, 0].min(1)).mean(),
      "first claim -> last fwd", (tp[:, :, 3].max(1) - tp[:, :, 0].min(1)).mean(),
      "last fwd -> first coef", (tp[:, :, 4].min(1) - tp[:, :, 3].max(1)).mean())
# throughput over time: rows whose backward finished per 50 us window
h, e = np.histogram(t[:, 6], bins=np.arange(0, t.max() + 50, 50))
print("rows done per 50us:", h.tolist())
h, e = np.histogram(t[:, 0], bins=np.arange(0, t.max() + 50, 50))
print("rows claimed per 50us:", h.tolist())
