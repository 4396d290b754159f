"""Run a few cfg-2 steps for profiling (ncu)."""
import sys
sys.path.insert(0, ".")
from paper_1909_13560_b200 import Solver, workloads as W
K = int(sys.argv[1]) if len(sys.argv) > 1 else 6
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
variant = int(sys.argv[3]) if len(sys.argv) > 3 else 0
with Solver(W.cfg2(K), kernel_variant=variant) as s:
    for _ in range(steps):
        s.step()
    s.layer(0)
