"""Build the sm_100a C-ABI library ``libhamming.so`` in-tree with nvcc.

``python -m paper_1412_6862_b200.build`` (or ``__graft_entry__.build()``).
Cross-compiles on a CPU-only box; the .so travels to the GPU box with the
repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SRC = os.path.join(PKG, "csrc", "hamming.cu")
HDR = os.path.join(ROOT, "include", "hamming.h")
LIB = os.path.join(PKG, "libhamming.so")

NVCC_FLAGS = [
    "-std=c++17", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "-Xptxas", "-v", "-diag-suppress", "177", "-Xcompiler", "-fPIC,-O2", "-shared",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    import glob
    deps = [SRC, HDR] + glob.glob(os.path.join(PKG, "csrc", "*.cuh"))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    if out == LIB and not force and not needs_build():
        return LIB
    tmp = out + f".tmp{os.getpid()}"
    cmd = [nvcc(), *NVCC_FLAGS, "-cudart", "static", *[f"-D{d}" for d in defines],
           "-I", os.path.join(ROOT, "include"), "-o", tmp, SRC]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libhamming.so")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", action="store_true")
    ap.add_argument("-o", default=LIB)
    ap.add_argument("-D", action="append", default=[])
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.v, out=a.o, defines=a.D))
