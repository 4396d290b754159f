"""Per-phase timing of the fused 1-D kernel (BSDE_PHASE_TIMING=1), cfg 2."""
import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, ".")
os.environ["BSDE_PHASE_TIMING"] = "1"
from paper_1909_13560_b200 import Solver, workloads as W, load_library
lib = load_library()
lib.bsde_internal_phase_times.argtypes = [C.c_void_p, C.POINTER(C.c_ulonglong), C.c_int]
variant = int(sys.argv[1]) if len(sys.argv) > 1 else 0
import time
t0 = time.time()
while time.time() - t0 < 2.0:                 # ramp the SM clock up before measuring
    with Solver(W.cfg2(6), kernel_variant=10 + variant) as s:
        s.solve()
names = ["start", "wait", "L1", "levels", "end", "Fs", "rhs", "pcr", "j1", "j2", "j3", "j4", "j5", "j6"]
for K in [1, 6]:
    with Solver(W.cfg2(K), kernel_variant=10 + variant) as s:
        for _ in range(20):
            s.step()
        nb = 147
        buf = (C.c_ulonglong * (16 * nb))()
        lib.bsde_internal_phase_times(s._h, buf, 16 * nb)
        a = np.array(buf, dtype=np.float64).reshape(nb, 16)
        a = a[a[:, 0] > 0]
        ref = a[:, 1:2]
        rel = (a - ref) / 1e3
        order = [0, 1, 5, 6, 7, 2, 8, 9, 10, 11, 12, 13, 3, 4]
        print(f"K={K}: " + "  ".join(f"{names[i]}={np.median(rel[:, i]):.2f}" for i in order if a[:, i].max() > 0), flush=True)
