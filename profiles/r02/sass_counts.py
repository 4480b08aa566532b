"""Count the Blackwell instructions that prove the hot path is hand-written sm_100a code
(UTCHMMA = tcgen05.mma, UTMALDG / UBLKCP = TMA, LDTM = tcgen05.ld, FFMA2/FADD2/FMUL2 = packed
fp32, MUFU.EX2) per kernel of the in-tree libodpo.so, and keep a short SASS excerpt."""
import collections
import re
import subprocess
import sys

so = sys.argv[1] if len(sys.argv) > 1 else "paper_2410_18252_b200/libodpo.so"
sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
OPS = ["UTCHMMA", "UTCBAR", "UTMALDG", "UBLKCP", "LDTM", "STTM", "FFMA2", "FADD2", "FMUL2", "MUFU.EX2",
       "LDG.E.NA.EFL2.256.CONSTANT", "STG.E.NA.EFL2.256"]
counts = collections.OrderedDict()
excerpt = collections.OrderedDict()
fn = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        fn = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        continue
    for op in OPS:
        if re.search(r"\b" + re.escape(op) + r"(\b|\s)", line):
            counts.setdefault(fn, collections.Counter())[op] += 1
            ex = excerpt.setdefault(fn, [])
            if len(ex) < 6 and not any(op in e for e in ex):
                ex.append(line.strip())
keep = ["k_engine<1, 0, 0, 1, odpo::Geo<4, 3, 4>", "k_row_bwd_split<1, 0, 512, 4, 32>",
        "k_engine<1, 1, 0, 1, odpo::Geo<4, 3, 4>", "k_engine<1, 2, 0, 1, odpo::Geo<8, 6, 2>",
        "k_lmhead_fwd2<false>", "k_lmhead_fwd2<true>", "k_gemm_tn2<false, true>",
        "k_gemm_tn2<true, true>", "k_vp_partials_warp<1>", "k_resident<1, 0, 0>"]
print("# SASS evidence: cuobjdump -sass of the in-tree libodpo.so (sm_100a)\n")
for k in keep:
    for f, c in counts.items():
        if k in f:
            print(f"## {f}")
            print("counts: " + ", ".join(f"{op} {c[op]}" for op in OPS if c[op]))
            print("```")
            print("\n".join(excerpt[f]))
            print("```\n")
            break
