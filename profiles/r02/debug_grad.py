"""Check of odpo_lmhead_grad's G scratch and both GEMMs (MN-major operands) against
torch on the GPU's own intermediates (debugging aid; tests/test_lmhead.py is the parity test)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import synth  # noqa: E402
import paper_2410_18252_b200 as odpo  # noqa: E402

R_T = [(11, 9), (40, 53)]
for (B, T), d, V, chunk in [((11, 9), 128, 1000, 256), ((40, 53), 256, 4133, 1024)]:
    R = B * T
    rows = np.arange(R)
    h, w = synth.lmhead_inputs(17, rows, d, V)
    tok = synth.tokens_rows(17, rows, V).reshape(B, T).astype(np.int32)
    mask = synth.mask_for(17, np.arange(B), T, "prefix", 3)
    hd = torch.from_numpy(h.reshape(B, T, d)).to(torch.bfloat16).cuda()
    wd = torch.from_numpy(w).to(torch.bfloat16).cuda()
    td, md = torch.from_numpy(tok).cuda(), torch.from_numpy(mask).cuda()
    ref = torch.full((B,), -30.0, device="cuda")
    pr = torch.arange(B - (B % 2), dtype=torch.int32, device="cuda").view(-1, 2)
    out = odpo.lmhead_online_dpo_loss_fwd(hd, wd, ref, td, md, 0.1, pair_rows=pr)
    L = odpo._L()
    CR = -(-min(chunk, R) // 256) * 256
    nb = L.odpo_lmhead_grad_scratch_bytes(CR, d, V)
    sc = torch.zeros(nb, dtype=torch.uint8, device="cuda")
    dh = torch.full((R, d), 7.0, device="cuda")
    dw = torch.full((V, d), 7.0, device="cuda")
    rc = L.odpo_lmhead_grad(C.c_void_p(hd.data_ptr()), C.c_void_p(wd.data_ptr()), R, d, V,
                            C.c_void_p(td.data_ptr()), C.c_void_p(out.row_lse.data_ptr()),
                            C.c_void_p(out.row_scale.data_ptr()), 1.0, C.c_void_p(dh.data_ptr()),
                            C.c_void_p(dw.data_ptr()), C.c_void_p(sc.data_ptr()), nb, CR, None)
    torch.cuda.synchronize()
    print("case", B, T, d, V, "chunk", CR, "rc", rc)
    Vp = -(-V // 8) * 8
    if R <= CR:
        G = sc[: 2 * CR * Vp].view(torch.bfloat16).float().view(CR, Vp)[:R, :V]
        print(" masked rows of G zero", bool((G[md.view(-1) == 0] == 0).all()),
              "rows with nonzero G", int((G.abs().sum(1) > 0).sum()), "/", R)
        dh_ref = G @ wd.float()
        dw_ref = G.t() @ hd.view(R, d).float()
        e1 = (dh - dh_ref).abs()
        e2 = (dw - dw_ref).abs()
        print(" dh max err", float(e1.max()), "at", np.unravel_index(int(e1.argmax()), tuple(e1.shape)),
              "rel", float(e1.max() / dh_ref.abs().max()))
        bad = (e1 > 1e-3 * dh_ref.abs().max()).nonzero()
        print("  bad dh rows", sorted(set(bad[:, 0].tolist()))[:20], "cols", sorted(set(bad[:, 1].tolist()))[:20])
        print(" dw max err", float(e2.max()), "rel", float(e2.max() / dw_ref.abs().max()))
        bad = (e2 > 1e-3 * dw_ref.abs().max()).nonzero()
        print("  bad dw rows", sorted(set(bad[:, 0].tolist()))[:20], "cols", sorted(set(bad[:, 1].tolist()))[:20])
