"""Per-phase breakdown of the persistent fused 1-D solve (BSDE_PHASE_TIMING=1, 32 stamps/step).
usage: python scripts/timeline2.py <kernel_variant> [K ...]"""
import ctypes as C, os, sys, time
import numpy as np
sys.path.insert(0, ".")
os.environ["BSDE_PHASE_TIMING"] = "1"
from paper_1909_13560_b200 import Solver, workloads as W, load_library
lib = load_library()
lib.bsde_internal_phase_times.argtypes = [C.c_void_p, C.POINTER(C.c_ulonglong), C.c_int]
kv = int(sys.argv[1]) if len(sys.argv) > 1 else 0
Ks = [int(x) for x in sys.argv[2:]] or [1, 6]
t0 = time.time()
while time.time() - t0 < 2.0:
    with Solver(W.cfg2(6)) as s:
        s.solve()
NAMES = {1: "ringwait+issue", 8: "red", 9: "epi", 10: "gap", 11: "donewait", 12: "vals", 13: "rhs",
         14: "pcr", 15: "c"}
for K in Ks:
    with Solver(W.cfg2(K), kernel_variant=kv) as s:
        nsteps = s.level
        s.solve()
        TP = {0: 224, 1: 448, 2: 480, 3: 480, 4: 224, 5: 320}[(kv % 100 - 10) if kv >= 10 else 0]
        nb = (65536 + TP - 1) // TP
        n = nsteps * nb * 32
        buf = (C.c_ulonglong * n)()
        lib.bsde_internal_phase_times(s._h, buf, n)
        a = np.array(buf, dtype=np.float64).reshape(nsteps, nb, 32) / 1e3
        a = a - a[0, :, 1].min()
        order = [0, 1] + [1 + j for j in range(K, 0, -1)] + [8, 9, 10, 11, 12, 13, 14, 15]
        order = [i for i in order if np.all(a[5:, :, i] > 0)]
        st = slice(20, nsteps - 5)
        end = a[:, :, 15]
        stepdur = np.diff(end.max(axis=1))[st]
        print(f"K={K} kv={kv} nb={nb}: step {np.median(stepdur):.2f} us (max-end diff);"
              f" per-CTA step {np.median(np.diff(end, axis=0)[st]):.2f}")
        parts = []
        for p_, i in zip(order[:-1], order[1:]):
            d = (a[:, :, i] - a[:, :, p_])[st]
            nm = NAMES.get(i, f"L{i - 1}")
            parts.append(f"{nm}={np.median(d):.2f}/{np.percentile(d, 90):.2f}")
        gap = (a[1:, :, 0] - a[:-1, :, 15])[st]
        print("   ", " ".join(parts), f"| loop={np.median(gap):.2f}")
        # per-CTA busy time (everything but the two neighbour waits), to find the pacing CTAs
        busy = (a[:, :, 15] - a[:, :, 0]) - (a[:, :, 1] - a[:, :, 0]) - (a[:, :, 11] - a[:, :, 10])
        bm = np.median(busy[st], axis=0)
        idx = np.argsort(bm)[::-1][:12]
        print("    busy median over CTAs %.2f us; slowest:" % np.median(bm),
              " ".join(f"{i}:{bm[i]:.2f}" for i in idx))
