"""Time bsde_solve_batch (cfg 2, K = 1..6) against six single persistent solves."""
import sys, time
sys.path.insert(0, ".")
from paper_1909_13560_b200 import Solver, solve_batch, workloads as W
kv = int(sys.argv[1]) if len(sys.argv) > 1 else 0
t0 = time.time()
while time.time() - t0 < 2.0:
    with Solver(W.cfg2(6)) as s:
        s.solve()
for rep in range(3):
    tot = 0.0
    for K in range(1, 7):
        with Solver(W.cfg2(K), kernel_variant=kv) as s:
            tot += s.solve().t_sweep_s
    ss = [Solver(W.cfg2(K), kernel_variant=kv) for K in range(1, 7)]
    r = solve_batch(ss)
    upd = sum(x.updates for x in r)
    print(f"kv={kv} singles {tot*1e3:.3f} ms ({upd/tot:.3e} upd/s)  batch {r[0].t_sweep_s*1e3:.3f} ms "
          f"({upd/r[0].t_sweep_s:.3e} upd/s)  y0 {[round(x.y0, 6) for x in r]}", flush=True)
    for s in ss:
        s.close()
