"""Build the CUDA library libbsde_b200.so in-tree (nvcc, sm_100a).

    python -m paper_1909_13560_b200.build
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libbsde_b200.so")
SOURCES = ["kernels.cu", "host.cu"]
HEADERS = ["bsde_internal.h", "problems.cuh", "fused1d.cuh", "fused1d_small.cuh", "fused2d.cuh", "fused3d.cuh",
           "aff2.cuh", "bicubic.cuh", "fsde.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]
LIBS = ["-L/usr/lib/x86_64-linux-gnu", "-lnccl"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "bsde.h"))
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    cmd = [NVCC, *FLAGS, "-o", LIB + ".tmp"] + [os.path.join(CSRC, f) for f in SOURCES] + LIBS
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libbsde_b200.so")
    with open(os.path.join(HERE, "ptxas_info.txt"), "w") as fh:
        fh.write(res.stderr)
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
