"""One persistent cfg-2 solve (for ncu)."""
import sys
sys.path.insert(0, ".")
from paper_1909_13560_b200 import Solver, workloads as W
K = int(sys.argv[1]) if len(sys.argv) > 1 else 6
with Solver(W.cfg2(K)) as s:
    s.solve()
