"""bsde_solve_batch (cfg 2, K = 1..6) per fused-kernel variant."""
import sys, time
sys.path.insert(0, ".")
from paper_1909_13560_b200 import Solver, solve_batch, workloads as W
vs = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0, 1, 4, 5]
t0 = time.time()
while time.time() - t0 < 2.0:
    with Solver(W.cfg2(6)) as s:
        s.solve()
for v in vs:
    best = 1e9
    for rep in range(2):
        ss = [Solver(W.cfg2(K), kernel_variant=10 + v) for K in range(1, 7)]
        try:
            r = solve_batch(ss)
            best = min(best, r[0].t_sweep_s)
            y0 = [round(x.y0, 6) for x in r]
        except Exception as e:
            print(f"variant {v}: {e}")
            best = None
            break
        finally:
            for s in ss:
                s.close()
    if best:
        print(f"variant {v}: batch {best*1e3:.3f} ms y0 {y0[:3]}", flush=True)
