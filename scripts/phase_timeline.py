"""Per-phase timeline of the fused 1-D kernel from the debug build's per-CTA %globaltimer stamps
(PHASE_STAMP in fused1d.cuh; libbsde_b200_debug.so built with -DBSDE_DEBUG by
`python scripts/phase_timeline.py --build`).  One single-problem solve of cfg 2 (K given), the
mean over CTAs and steps of the time between consecutive stamps of pass 1 / pass 2.
usage: BSDE_PHASE_TIMING=1 python scripts/phase_timeline.py K [variant]"""
import ctypes as C
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
DBG = os.path.join(ROOT, "paper_1909_13560_b200", "libbsde_b200_debug.so")

if "--build" in sys.argv:
    from paper_1909_13560_b200 import build as b
    cmd = [b.NVCC, *b.FLAGS, "-DBSDE_DEBUG", "-o", DBG] + [os.path.join(b.CSRC, f) for f in b.SOURCES] + b.LIBS
    subprocess.run(cmd, check=True, capture_output=True)
    sys.exit(0)

from paper_1909_13560_b200 import bsde  # noqa: E402
lib = bsde.load_library(DBG)
lib.bsde_internal_phase_times.argtypes = [C.c_void_p, C.POINTER(C.c_ulonglong), C.c_int]
from paper_1909_13560_b200 import Solver, workloads as W  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 6
variant = int(sys.argv[2]) if len(sys.argv) > 2 else 0
blocks = int(sys.argv[3]) if len(sys.argv) > 3 else 293          # CTAs of the launch (stamp stride)
with Solver(W.cfg2(K), kernel_variant=10 + variant) as s:
    r = s.solve()
    n = 600 * 1100 * 32
    buf = (C.c_ulonglong * n)()
    lib.bsde_internal_phase_times(s._h, buf, n)
    a = np.frombuffer(buf, dtype=np.uint64)[:600 * blocks * 32].reshape(600, blocks, 32).astype(np.float64)
steps = 257 - K
a = a[5:steps - 5]                                   # steady state
print(f"K={K} variant={variant}: sweep {r.t_sweep_s * 1e3:.3f} ms, {blocks} CTAs, {r.t_sweep_s / steps * 1e6:.2f} us/step")
order = [0, 1] + [1 + j for j in range(K, 0, -1)] + [8, 16, 17, 18, 9, 10, 11, 12, 13, 14, 15]
names = {0: "start", 1: "taps", 8: "red.write", 16: "red.read", 17: "prefetch", 18: "epilogue", 9: "done.flag",
         10: "p2.start", 11: "p2.flags", 12: "p2.values", 13: "p2.rhs", 14: "p2.pcr", 15: "p2.coef"}
prev = order[0]
for i in order[1:]:
    d = (a[:, :, i] - a[:, :, prev]) / 1e3
    print(f"  {names.get(prev, f'lvl{prev - 1}'):>10} -> {names.get(i, f'lvl{i - 1}'):<10} mean {np.mean(d):7.3f} us   p90 {np.percentile(d, 90):7.3f}")
    prev = i
nxt = (a[1:, :, 0] - a[:-1, :, 15]) / 1e3
print(f"  {'p2.coef':>10} -> {'next start':<10} mean {np.mean(nxt):7.3f} us")
print(f"  step (start -> next start) mean {np.mean((a[1:, :, 0] - a[:-1, :, 0]) / 1e3):.3f} us")
print(f"  max over CTAs of epilogue -> done.flag: mean {np.mean(np.max(a[:, :, 9] - a[:, :, 18], axis=1)) / 1e3:.3f} us")
