"""Tuning builds of libodpo.so with alternative geometry-1 shapes (ODPO_G1_NCW/STAGES/CPS), for
profiles/tune_geo1.sh.  Output: build_variants/libodpo_g1_<ncw>_<stages>_<cps>.so (git-ignored)."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_18252_b200 import build as b  # noqa: E402

VARIANTS = [tuple(int(x) for x in v.split(",")) for v in sys.argv[1:]] or [
    (16, 12, 1), (8, 12, 1), (16, 8, 1), (8, 10, 1)]


def one(v):
    ncw, st, cps = v
    out = os.path.join(ROOT, "build_variants", f"libodpo_g1_{ncw}_{st}_{cps}.so")
    b.build(force=True, out=out, defines={"ODPO_G1_NCW": ncw, "ODPO_G1_STAGES": st, "ODPO_G1_CPS": cps})
    return out


os.makedirs(os.path.join(ROOT, "build_variants"), exist_ok=True)
with ThreadPoolExecutor(4) as ex:
    for o in ex.map(one, VARIANTS):
        print(o)
