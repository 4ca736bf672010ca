"""Build libswx.so (sm_100a) in-tree with nvcc.

    python -m paper_1805_06557_b200.build

Produces ``paper_1805_06557_b200/libswx.so``; the .so is git-ignored but
travels to the GPU box with the gpurun snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libswx.so")
SOURCES = ["rexi.cu", "sht.cu", "host.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "swx.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, trace: bool = False) -> str:
    """trace=True compiles the per-CTA phase marks read by swx_trace."""
    if not force and not stale():
        return LIB
    cuda = os.path.dirname(os.path.dirname(nvcc()))
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "--shared",
           "-Xcompiler", "-fPIC", "-Xcompiler", "-fopenmp", "-Xptxas", "-warn-spills",
           *[os.path.join(CSRC, s) for s in SOURCES],
           *(["-DSWX_TRACE"] if trace else []),
           *[f"-D{d}" for d in os.environ.get("SWX_DEFINES", "").split()],
           "-o", LIB + ".tmp",
           f"-L{cuda}/lib64", "-lcufft", "-lgomp", f"-Xlinker", f"-rpath={cuda}/lib64"]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv or "--trace" in sys.argv, verbose=True,
          trace="--trace" in sys.argv)
    print(LIB)
