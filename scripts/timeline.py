"""Per-step, per-CTA phase timeline of a persistent fused solve (BSDE_PHASE_TIMING=1)."""
import ctypes as C, os, sys, time
import numpy as np
sys.path.insert(0, ".")
os.environ["BSDE_PHASE_TIMING"] = "1"
from paper_1909_13560_b200 import Solver, workloads as W, load_library
lib = load_library()
lib.bsde_internal_phase_times.argtypes = [C.c_void_p, C.POINTER(C.c_ulonglong), C.c_int]
variant = int(sys.argv[1]) if len(sys.argv) > 1 else 0
t0 = time.time()
while time.time() - t0 < 2.0:
    with Solver(W.cfg2(6)) as s:
        s.solve()
for K in [1, 6]:
    with Solver(W.cfg2(K), kernel_variant=10 + variant) as s:
        nsteps = s.level
        s.solve()
        P = 65536
        TP = {0: 224, 1: 448, 2: 480, 3: 480, 4: 224, 5: 320}[variant]
        nb = (P + TP - 1) // TP
        n = nsteps * nb * 16
        buf = (C.c_ulonglong * n)()
        lib.bsde_internal_phase_times(s._h, buf, n)
        a = np.array(buf, dtype=np.float64).reshape(nsteps, nb, 16) / 1e3
        t00 = a[0, :, 1].min()
        a = a - t00
        # per-step: end times (stamp 4) distribution and per-phase medians
        st = slice(20, nsteps - 5)
        end = a[:, :, 4]
        stepdur = np.diff(end.max(axis=1))[st]
        print(f"K={K} variant={variant} nb={nb} steps={nsteps}: step (max end diff) median {np.median(stepdur):.2f} us")
        names = {2: "issue", 5: "rhs", 6: "pcr", 7: "c+flag", 8: "L1", 3: "lv", 4: "epi"}
        for j in range(K, 1, -1):
            names[7 + j] = f"L{j}"
        order = [2] + [7 + j for j in range(K, 1, -1)] + [5, 6, 7, 8, 3, 4]
        prev = 2
        parts = []
        for i in order[1:]:
            parts.append(f"{names[i]}={np.median((a[:, :, i] - a[:, :, prev])[st]):.2f}")
            prev = i
        # start of step (stamp 2) relative to previous end
        gap = (a[1:, :, 2] - a[:-1, :, 4])[st]
        print("   ", " ".join(parts), f" | start-after-prev-end={np.median(gap):.2f}")
        # skew across CTAs within a step
        print(f"    end skew within step: median {np.median((end.max(1)-end.min(1))[st]):.2f} us; slowest CTA ids:",
              np.bincount(np.argmax(end[st], axis=1), minlength=nb).argsort()[-5:])
