"""Per-round timeline of the batched fused 1-D launch (cfg 2, K = 1..6) from the debug build's
%globaltimer stamps (PHASE_STAMP in fused1d.cuh; build libbsde_b200_debug.so with
`python scripts/phase_timeline.py --build`).  Per problem (its own CTAs in the partitioned
schedule): round time, pass 1 (all tiles), the pass-2 flag wait and the pass-2 spline.
usage: BSDE_PHASE_TIMING=1 python scripts/batch_timeline.py [grid CTAs (pairs: half the sum)]"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
DBG = os.path.join(ROOT, "paper_1909_13560_b200", "libbsde_b200_debug.so")
from paper_1909_13560_b200 import bsde  # noqa: E402
lib = bsde.load_library(DBG)
lib.bsde_internal_phase_times.argtypes = [C.c_void_p, C.POINTER(C.c_ulonglong), C.c_int]
from paper_1909_13560_b200 import Solver, solve_batch, workloads as W  # noqa: E402

ss = [Solver(W.cfg2(K)) for K in range(1, 7)]
res = solve_batch(ss)
nb = int(sys.argv[1]) if len(sys.argv) > 1 else sum(r.batch_ctas for r in res)   # the launch's grid
print(f"batch {res[0].t_sweep_s * 1e3:.3f} ms, {nb} CTAs")
for K, s, r in zip(range(1, 7), ss, res):
    n = 600 * 1100 * 32
    buf = (C.c_ulonglong * n)()
    lib.bsde_internal_phase_times(s._h, buf, n)
    a = np.frombuffer(buf, dtype=np.uint64)[:600 * nb * 32].reshape(600, nb, 32).astype(np.float64)
    steps = 257 - K
    used = np.nonzero(a[10, :, 20])[0]                    # this problem's CTAs
    a = a[5:steps - 5][:, used]                          # steady state
    rnd = (a[1:, :, 20] - a[:-1, :, 20]) / 1e3
    p1 = (a[:, :, 9] - a[:, :, 20]) / 1e3
    w2 = (a[:, :, 11] - a[:, :, 10]) / 1e3
    s2 = (a[:, :, 15] - a[:, :, 11]) / 1e3
    lv = (a[:, :, 8] - a[:, :, 1]) / 1e3                  # last unit: taps -> reduction (levels)
    ep = (a[:, :, 9] - a[:, :, 8]) / 1e3                  # last unit: reduction + epilogue
    ph = [np.mean((a[:, :, i + 1] - a[:, :, i]) / 1e3) for i in (11, 12, 13, 14)]
    print(f"K={K}: {r.batch_ctas} CTAs x {r.batch_tiles} tiles: round {np.mean(rnd):6.2f} us | pass1 {np.mean(p1):6.2f} "
          f"(last tile: levels {np.mean(lv):5.2f}, epilogue {np.mean(ep):5.2f}) | p2 wait {np.mean(w2):5.2f} "
          f"p2 spline {np.mean(s2):5.2f} (values {ph[0]:4.2f} rhs {ph[1]:4.2f} filter {ph[2]:4.2f} coef {ph[3]:4.2f})"
          f" | p90 round {np.percentile(rnd, 90):6.2f}")
for s in ss:
    s.close()
