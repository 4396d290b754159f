"""Time the fused 1-D kernel variants on cfg 2 (K = 1, 3, 6) and check they agree."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1909_13560_b200 import Solver, workloads as W

nv = int(sys.argv[1]) if len(sys.argv) > 1 else 6
vlist = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else list(range(nv))
ref = {}
import time
t0 = time.time()
while time.time() - t0 < 2.0:                 # ramp the SM clock up before measuring
    with Solver(W.cfg2(6)) as s:
        s.solve()
for K in [1, 3, 6]:
    for v in vlist:
        ts = []
        for rep in range(3):
            with Solver(W.cfg2(K), kernel_variant=10 + v) as s:
                r = s.solve()
                ts.append(r.t_sweep_s)
                lay = s.layers()
        if v == vlist[0]:
            ref[K] = lay
        err = float(np.max(np.abs(lay - ref[K]) / np.max(np.abs(ref[K]), axis=1, keepdims=True)))
        steps = 256 - K + 1
        print(f"K={K} variant={v} sweep_ms={min(ts)*1e3:.3f} us_per_step={min(ts)/steps*1e6:.2f} "
              f"upd/s={65536*steps/min(ts):.3e} rel_vs_v0={err:.2e}", flush=True)
