"""Per-phase breakdown of bsde_solve_batch over cfg 2 K = 1..6 (BSDE_PHASE_TIMING=1)."""
import ctypes as C, os, sys, time
import numpy as np
sys.path.insert(0, ".")
os.environ["BSDE_PHASE_TIMING"] = "1"
from paper_1909_13560_b200 import Solver, solve_batch, workloads as W, load_library
lib = load_library()
lib.bsde_internal_phase_times.argtypes = [C.c_void_p, C.POINTER(C.c_ulonglong), C.c_int]
Ks = [int(x) for x in sys.argv[1:]] or [1, 2, 3, 4, 5, 6]
t0 = time.time()
while time.time() - t0 < 2.0:
    with Solver(W.cfg2(6)) as s:
        s.solve()
ss = [Solver(W.cfg2(K)) for K in Ks]
steps = [s.level for s in ss]
r = solve_batch(ss)
print(f"batch {r[0].t_sweep_s*1e3:.3f} ms")
nb = (65536 + 223) // 224
A = []
for s, ns in zip(ss, steps):
    n = ns * nb * 32
    buf = (C.c_ulonglong * n)()
    lib.bsde_internal_phase_times(s._h, buf, n)
    A.append(np.array(buf, dtype=np.float64).reshape(ns, nb, 32) / 1e3)
t00 = min(a[0, :, 0].min() for a in A)
NAMES = {1: "wait+issue", 8: "red", 9: "epi", 10: "->p2", 11: "donewait", 12: "vals", 13: "rhs", 14: "pcr", 15: "c"}
st = slice(20, min(steps) - 5)
for K, a in zip(Ks, A):
    a = a - t00
    order = [0, 1] + [1 + j for j in range(K, 0, -1)] + [8, 9, 10, 11, 12, 13, 14, 15]
    parts = []
    for p_, i in zip(order[:-1], order[1:]):
        d = (a[:, :, i] - a[:, :, p_])[st]
        parts.append(f"{NAMES.get(i, f'L{i - 1}')}={np.median(d):.2f}")
    rd = np.diff(a[:, :, 0], axis=0)[st]
    print(f"K={K}: round {np.median(rd):.2f} us |", " ".join(parts))
# order within a round: gaps between problems' pass-1 ends and the next's start
ends = [a[:, :, 9] for a in A]
starts = [a[:, :, 0] for a in A]
for i in range(len(A) - 1):
    m = min(len(starts[i + 1]), len(ends[i]))
    print(f"p1 gap {Ks[i]}->{Ks[i+1]}: {np.median((starts[i+1][:m] - ends[i][:m])[st]):.2f} us")
m = min(len(A[0]), len(ends[-1]))
print(f"p1 end -> p2 start: {np.median((A[0][:m, :, 10] - ends[-1][:m])[st]):.2f} us")
for s in ss:
    s.close()
