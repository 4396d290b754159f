"""One bsde_solve_batch over cfg 2 K = 1..6 (for ncu: the launch bench.py times)."""
import sys
sys.path.insert(0, ".")
from paper_1909_13560_b200 import Solver, solve_batch, workloads as W
ss = [Solver(W.cfg2(K)) for K in range(1, 7)]
solve_batch(ss)
for s in ss:
    s.close()
