"""Chronological phase stamps of one round of bsde_solve_batch (cfg 2, K = 1..6), medians over
rounds 20..end-5 and all CTAs, relative to the round start (BSDE_PHASE_TIMING=1)."""
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
m = min(steps)
rounds = range(20, m - 5)
start = np.min([a[:m, :, 0] for a in A], axis=0)          # round start per (round, CTA)
NAMES = {0: "p1 start", 1: "windows issued", 8: "levels done", 9: "epilogue done", 10: "p2 start",
         11: "done flags ok", 12: "values in", 13: "rhs", 14: "pcr", 15: "coefs stored", 16: "red read", 17: "next windows issued", 18: "picard+stores (warp 0)"}
ev = []
for K, a in zip(Ks, A):
    for i in range(32):
        v = a[:m, :, i]
        if not np.any(v[rounds] > 0):
            continue
        rel = (v - start)[rounds]
        name = NAMES.get(i, f"L{i - 1} done" if 2 <= i <= 7 else f"#{i}")
        ev.append((float(np.median(rel)), f"K={K} {name}"))
ev.sort()
prev = 0.0
for t, name in ev:
    print(f"{t:8.2f} us (+{t - prev:5.2f})  {name}")
    prev = t
rd = np.diff(start, axis=0)[rounds]
print(f"round {np.median(rd):.2f} us")
for s in ss:
    s.close()
