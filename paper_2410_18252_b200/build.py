"""Build libodpo.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libodpo.so")
SOURCES = [os.path.join(CSRC, "odpo.cu"), os.path.join(CSRC, "odpo_lmhead.cu")]
DEPS = SOURCES + [os.path.join(CSRC, "odpo_device.cuh"), os.path.join(CSRC, "odpo_engine.cuh"), os.path.join(CSRC, "odpo_resident.cuh"),
                  os.path.join(ROOT, "include", "odpo.h")]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: dict | None = None) -> str:
    lib = out or LIB
    stale = force or not os.path.exists(lib) or any(
        os.path.getmtime(lib) < os.path.getmtime(d) for d in DEPS)
    if stale:
        dflags = [f"-D{k}={v}" for k, v in (defines or {}).items()]
        cmd = ["nvcc", *NVCC_FLAGS, *dflags, "-I", os.path.join(ROOT, "include"), "-o", lib, *SOURCES]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{res.stdout}\n{res.stderr}")
        if verbose:
            print(res.stderr)
    return lib


if __name__ == "__main__":
    print(build(force=True, verbose=True))
