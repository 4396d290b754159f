import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1909_13560_b200 import Solver, workloads as W
for spec in [W.ex4_2d(3, 6, npts=33), W.ex4_2d(3, 8, npts=257), W.ex4_2d(1, 4, npts=24)]:
    a = Solver(spec, kernel_variant=0); b = Solver(spec, kernel_variant=1)
    a.step(); b.step()
    torch.cuda.synchronize()
    for f in range(3):
        la, lb = a.layer(f), b.layer(f)
        d = np.abs(la - lb)
        i = np.unravel_index(np.argmax(d), d.shape)
        print(spec["name"], spec["npts"], "field", f, "maxdiff", d.max(), "at", i, la[i], lb[i], "mean |a|", np.abs(la).mean(), flush=True)
    print("launches", a.kernel_launches, b.kernel_launches)
