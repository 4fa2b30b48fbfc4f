"""In-tree build of the sm_100a CUDA library (libwhb200.so).

The built .so lives next to the package (git-ignored, but it travels to the
GPU box with the gpurun snapshot).  nvcc cross-compiles here without a GPU.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SRC = os.path.join(PKG, "csrc", "whb200.cu")
LIB_DIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIB_DIR, "libwhb200.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",                 # no FMA contraction: bitwise parity with the reference
    "-Xptxas", "-v",
    "-shared", "-Xcompiler", "-fPIC",
    "-I", os.path.join(ROOT, "include"),
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [SRC, os.path.join(ROOT, "include", "whb200.h")]
    deps += [os.path.join(PKG, "csrc", f) for f in os.listdir(os.path.join(PKG, "csrc"))]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def source_sha16() -> str:
    """sha256 (16 hex digits) of everything the library is built from: the CUDA sources, the
    public header and the nvcc flags.  nvcc's output is not byte-reproducible (it embeds
    per-compile module ids), so measurements are tied to the build inputs instead."""
    import hashlib

    # (flags without the checkout's absolute include path: the same sources hash the same anywhere)
    h = hashlib.sha256(" ".join(f for f in NVCC_FLAGS if not f.startswith(ROOT)).encode())
    csrc = os.path.join(PKG, "csrc")
    for fn in sorted(os.listdir(csrc)):
        if fn.endswith((".cu", ".cuh", ".h")):
            h.update(fn.encode())
            h.update(open(os.path.join(csrc, fn), "rb").read())
    h.update(open(os.path.join(ROOT, "include", "whb200.h"), "rb").read())
    return h.hexdigest()[:16]


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    os.makedirs(LIB_DIR, exist_ok=True)
    tmp = LIB + ".tmp"
    cmd = [nvcc(), *NVCC_FLAGS, "-o", tmp, SRC]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = r.stdout + r.stderr
    with open(os.path.join(LIB_DIR, "build.log"), "w") as fh:
        fh.write(" ".join(cmd) + "\n" + log)
    if r.returncode != 0:
        sys.stderr.write(log)
        raise RuntimeError(f"nvcc failed ({r.returncode}); see {LIB_DIR}/build.log")
    if verbose:
        sys.stderr.write(log)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
