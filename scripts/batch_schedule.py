"""Device time of the cfg 2 batch (K = 1..6) per CTA schedule: round robin (mode 1), the
planned partition (mode 2) and forced tiles-per-CTA ns = 1..8 (modes 11..18); and single
problems with forced ns (the cost-model calibration of host.cu plan_batch_partition)."""
import sys
import time
sys.path.insert(0, ".")
from paper_1909_13560_b200 import Solver, solve_batch, workloads as W  # noqa: E402

t0 = time.time()
while time.time() - t0 < 2.0:
    with Solver(W.cfg2(6)) as s:
        s.solve()


def run(Ks, mode, reps=2):
    best, sched = 1e9, None
    for _ in range(reps):
        ss = [Solver(W.cfg2(K)) for K in Ks]
        try:
            r = solve_batch(ss, mode=mode)
            if r[0].t_sweep_s < best:
                best, sched = r[0].t_sweep_s, [(x.batch_ctas, x.batch_tiles) for x in r]
        except Exception as exc:  # noqa: BLE001 -- infeasible forced schedules
            return float("nan"), str(exc)[:60]
        finally:
            for s in ss:
                s.close()
    return best, sched


for mode in [3, 2, 1, 0]:
    t, sc = run(range(1, 7), mode)
    print(f"batch K=1..6 mode {mode}: {t * 1e3:.3f} ms  schedule {sc}", flush=True)
for K in (1, 6):
    for mode in [11, 12, 14]:
        t, sc = run([K], mode)
        print(f"single K={K} mode {mode}: {t * 1e3:.3f} ms ({t / (257 - K) * 1e6:.2f} us/step) schedule {sc}", flush=True)
