"""Busy time of the batched cfg-2 launch: the same launch with every neighbour-flag wait
skipped (BSDE_DEBUG_NOWAIT: results are wrong, timing only), per-CTA mean round time."""
import ctypes as C, os, sys, time
import numpy as np
sys.path.insert(0, ".")
os.environ["BSDE_PHASE_TIMING"] = "1"
from paper_1909_13560_b200 import Solver, solve_batch, workloads as W, load_library
lib = load_library()
lib.bsde_internal_phase_times.argtypes = [C.c_void_p, C.POINTER(C.c_ulonglong), C.c_int]
t0 = time.time()
while time.time() - t0 < 2.0:
    with Solver(W.cfg2(6)) as s:
        s.solve()
for mode in ["wait", "nowait", "nowait+nopad"]:
    for k, on in (("BSDE_DEBUG_NOWAIT", "nowait" in mode), ("BSDE_DEBUG_NOPAD", "nopad" in mode)):
        if on:
            os.environ[k] = "1"
        else:
            os.environ.pop(k, None)
    ss = [Solver(W.cfg2(K)) for K in range(1, 7)]
    steps = [s.level for s in ss]
    r = solve_batch(ss)
    nb = (65536 + 223) // 224
    A = []
    for s, ns in zip(ss, steps):
        n = ns * nb * 32
        buf = (C.c_ulonglong * n)()
        lib.bsde_internal_phase_times(s._h, buf, n)
        A.append(np.array(buf, dtype=np.float64).reshape(ns, nb, 32) / 1e3)
    m = min(steps)
    start = np.min([a[:m, :, 0] for a in A], axis=0)
    rd = np.diff(start, axis=0)[20:m - 5]          # (rounds, CTAs)
    per_cta = rd.mean(axis=0)
    order = np.argsort(per_cta)
    print(f"{mode}: batch {r[0].t_sweep_s*1e3:.3f} ms, round median {np.median(rd):.2f} us, per-CTA mean round "
          f"min {per_cta.min():.2f} (CTA {order[0]}) max {per_cta.max():.2f} (CTA {order[-1]}); slowest CTAs "
          f"{list(order[-6:][::-1])}; first/last CTA {per_cta[0]:.2f}/{per_cta[-1]:.2f}", flush=True)
    for s in ss:
        s.close()

# per-phase durations (nowait launch) of selected CTAs: the edges, an interior CTA
os.environ["BSDE_DEBUG_NOWAIT"] = "1"
os.environ["BSDE_DEBUG_NOPAD"] = "1"
ss = [Solver(W.cfg2(K)) for K in range(1, 7)]
steps = [s.level for s in ss]
solve_batch(ss)
nb = (65536 + 223) // 224
A = []
for s, ns in zip(ss, steps):
    n = ns * nb * 32
    buf = (C.c_ulonglong * n)()
    lib.bsde_internal_phase_times(s._h, buf, n)
    A.append(np.array(buf, dtype=np.float64).reshape(ns, nb, 32) / 1e3)
m = min(steps)
sel = [0, 1, 146, 291, 292]
NAMES = {0: "p1", 1: "win", 8: "lev", 9: "epi", 10: "p2", 11: "dw", 12: "val", 13: "rhs", 14: "pcr", 15: "c",
         16: "red", 17: "nwin", 18: "pic"}
for K, a in zip(range(1, 7), A):
    order = [0, 1] + [1 + j for j in range(K, 0, -1)] + [8, 16, 17, 18, 9, 10, 11, 12, 13, 14, 15]
    for cta in sel:
        parts = []
        for p_, i in zip(order[:-1], order[1:]):
            d = (a[20:m - 5, cta, i] - a[20:m - 5, cta, p_])
            parts.append(f"{NAMES.get(i, f'L{i - 1}')}={np.median(d):.2f}")
        print(f"K={K} CTA {cta:3d}: " + " ".join(parts))
for s in ss:
    s.close()
