"""cfg 4: setup + a few steps (for ncu)."""
import sys
sys.path.insert(0, ".")
from paper_1909_13560_b200 import Solver, workloads as W
P = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
with Solver(W.cfg4(P)) as s:
    for _ in range(steps):
        s.step()
    s.layer(0)
