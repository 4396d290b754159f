"""Per-CTA end times of one fused step (edge CTAs vs median) -- BSDE_PHASE_TIMING=1."""
import ctypes as C, os, sys, time
import numpy as np
sys.path.insert(0, ".")
os.environ["BSDE_PHASE_TIMING"] = "1"
from paper_1909_13560_b200 import Solver, workloads as W, load_library
lib = load_library()
lib.bsde_internal_phase_times.argtypes = [C.c_void_p, C.POINTER(C.c_ulonglong), C.c_int]
t0 = time.time()
while time.time() - t0 < 2.0:
    with Solver(W.cfg2(6)) as s:
        s.solve()
for K in [1, 6]:
    with Solver(W.cfg2(K)) as s:
        for _ in range(20):
            s.step()
        nb = 147
        buf = (C.c_ulonglong * (16 * nb))()
        lib.bsde_internal_phase_times(s._h, buf, 16 * nb)
        a = np.array(buf, dtype=np.float64).reshape(nb, 16)
        a = a[a[:, 0] > 0]
        rel = (a - a[:, 1:2]) / 1e3
        dur = rel[:, 4]
        print(f"K={K} nCTA={len(a)} step(wait->end) median {np.median(dur):.2f} min {dur.min():.2f} max {dur.max():.2f} "
              f"CTA0 {dur[0]:.2f} CTA1 {dur[1]:.2f} CTA2 {dur[2]:.2f} last {dur[-1]:.2f} last-1 {dur[-2]:.2f}")
        print("   spline(7-1):", np.round(rel[[0, 1, 2, len(a)//2, -2, -1], 7], 2), " levels(3-7):",
              np.round((rel[:, 3] - rel[:, 7])[[0, 1, 2, len(a)//2, -2, -1]], 2))
        start_abs = a[:, 0] - a[:, 0].min()
        wait_abs = a[:, 1] - a[:, 0].min()
        end_abs = a[:, 4] - a[:, 0].min()
        print(f"   abs: start spread {start_abs.min()/1e3:.2f}..{start_abs.max()/1e3:.2f}  wait release {wait_abs.min()/1e3:.2f}..{wait_abs.max()/1e3:.2f}  end {end_abs.min()/1e3:.2f}..{end_abs.max()/1e3:.2f} us")
