"""Device time of single cfg 2 solves per K and of the batched launch per fused-kernel variant
(the breakdown behind DESIGN.md §5).  usage: python scripts/k_sweep.py [variants]"""
import sys
import time
sys.path.insert(0, ".")
from paper_1909_13560_b200 import Solver, solve_batch, workloads as W  # noqa: E402

vs = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0]
t0 = time.time()
while time.time() - t0 < 2.0:                  # clocks up
    with Solver(W.cfg2(6)) as s:
        s.solve()
for v in vs:
    for K in range(1, 7):
        best = 1e9
        for _ in range(3):
            with Solver(W.cfg2(K), kernel_variant=10 + v) as s:
                r = s.solve()
                best = min(best, r.t_sweep_s)
        print(f"variant {v} K={K}: {best * 1e3:.3f} ms ({(257 - K) / best / 1e3:.1f} steps/ms)", flush=True)
    for mode in (1, 2):
        best = 1e9
        for _ in range(3):
            ss = [Solver(W.cfg2(K), kernel_variant=10 + v) for K in range(1, 7)]
            try:
                r = solve_batch(ss, mode=mode)
                best = min(best, r[0].t_sweep_s)
            except Exception as exc:  # noqa: BLE001
                print(f"variant {v} mode {mode}: {exc}")
                best = None
                break
            finally:
                for s in ss:
                    s.close()
        if best:
            print(f"variant {v} batch K=1..6 mode {mode}: {best * 1e3:.3f} ms", flush=True)
