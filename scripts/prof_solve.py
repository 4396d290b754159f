"""One persistent cfg-2 solve (for ncu).  usage: prof_solve.py K [kernel_variant]"""
import sys
sys.path.insert(0, ".")
from paper_1909_13560_b200 import Solver, workloads as W
K = int(sys.argv[1]) if len(sys.argv) > 1 else 6
kv = int(sys.argv[2]) if len(sys.argv) > 2 else 0
with Solver(W.cfg2(K), kernel_variant=kv) as s:
    s.solve()
