"""Sub-phase medians of one fused step (BSDE_PHASE_TIMING=1)."""
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
names = {1: "wait", 2: "issue", 5: "rhs", 6: "pcr", 7: "c+flag", 13: "j6", 12: "j5", 11: "j4", 10: "j3", 9: "j2", 8: "j1", 3: "lv", 4: "epi"}
for K in [1, 6]:
    for mode in ["step", "solve"]:
        with Solver(W.cfg2(K)) as s:
            if mode == "step":
                for _ in range(20):
                    s.step()
            else:
                s.solve()
            nb = 147
            buf = (C.c_ulonglong * (16 * nb))()
            lib.bsde_internal_phase_times(s._h, buf, 16 * nb)
            a = np.array(buf, dtype=np.float64).reshape(nb, 16)
            a = a[a[:, 0] > 0]
            order = [1, 2] + [7 + j for j in range(K, 1, -1)] + [5, 6, 7, 8, 3, 4]
            out = []
            prev = order[0]
            for i in order[1:]:
                out.append(f"{names[i]}={np.median(a[:, i] - a[:, prev]) / 1e3:.2f}")
                prev = i
            print(f"K={K} {mode}: " + " ".join(out) + f"  | total={np.median(a[:, 4] - a[:, 1]) / 1e3:.2f}", flush=True)
