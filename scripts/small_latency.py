"""Wall time of bsde_setup + bsde_solve for small Ex. 1 problems (the TTS sweep's cheap end)."""
import sys, time
sys.path.insert(0, ".")
from paper_1909_13560_b200 import Solver, workloads as W
with Solver(W.ex1(3, 64)) as s:
    s.solve()
for K, N in [(2, 16), (2, 16), (5, 64), (5, 64), (1, 16)]:
    t0 = time.perf_counter()
    s = Solver(W.ex1(K, N))
    t1 = time.perf_counter()
    r = s.solve()
    t2 = time.perf_counter()
    shape, nl = s.shape, s.kernel_launches
    s.close()
    t3 = time.perf_counter()
    print(f"K={K} N={N} P={shape[0]} setup {1e3*(t1-t0):.2f} ms solve {1e3*(t2-t1):.2f} ms close {1e3*(t3-t2):.2f} ms launches {nl}")
