"""Run the CPU oracle on every printed error row of Tables 4, 5 and 9 (tests/golden/
printed_tables.txt) and print measured/printed ratios.  Used to decide, per row, whether the
row is a gated pin or excluded (R10 for K = 2, the rounding floor, runtime).

    python scripts/printed_rows.py [max_cost]      (cost ~ points x steps x K x L^d)
"""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import oracle  # noqa: E402
from paper_1909_13560_b200 import workloads as W  # noqa: E402

max_cost = float(sys.argv[1]) if len(sys.argv) > 1 else 4e10
rows = [ln.split() for ln in open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "printed_tables.txt"))
        if ln.strip() and not ln.startswith("#")]
for r in rows:
    ex, K, N, M, ye, ze = r[0], int(r[1]), int(r[2]), int(r[3]), float(r[4]), float(r[5])
    d = 2 if ex == "ex4" else 1
    L = 8 if d == 2 else 32
    cost = float(M + 1) ** d * N * K * L ** d
    if cost > max_cost:
        print(f"{ex} K={K} N={N} M={M}: skipped (cost {cost:.1e})", flush=True)
        continue
    spec = {"ex1": W.ex1, "ex2": W.ex2, "ex4": W.ex4_2d}[ex](K, N)
    t0 = time.time()
    o = oracle.Oracle(spec, nthreads=os.cpu_count())
    y0, z0 = o.solve()
    o.close()
    ref = W.reference_solution(spec)
    ey = abs(y0 - ref[0])
    ez = float(np.sqrt(sum((z0[k] - ref[1][k]) ** 2 for k in range(d))))
    print(f"{ex} K={K} N={N} M={M}: y {ey:.3e} / {ye:.2e} = {ey / ye:.3f}   z {ez:.3e} / {ze:.2e} = {ez / ze:.3f}"
          f"   ({time.time() - t0:.1f} s)", flush=True)
