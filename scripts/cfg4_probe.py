"""Time a few cfg-4 steps (2-D exchange, 4096^2, K=4, L=8) with the generic kernel."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import torch
from paper_1909_13560_b200 import Solver, workloads as W
P = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
spec = W.cfg4(P)
t0 = time.time()
variant = int(sys.argv[3]) if len(sys.argv) > 3 else 0
ts = torch.cuda.Stream()
torch.cuda.set_stream(ts)
s = Solver(spec, stream=ts.cuda_stream, kernel_variant=variant)
torch.cuda.synchronize()
print("setup s", time.time() - t0, "shape", s.shape, flush=True)
for rep in range(2):
    st = torch.cuda.Event(enable_timing=True); en = torch.cuda.Event(enable_timing=True)
    st.record(ts)
    for _ in range(steps):
        s.step()
    en.record(ts); torch.cuda.synchronize()
    ms = st.elapsed_time(en) / steps
    print(f"P={P} per-step {ms:.3f} ms  -> {P*P/ms*1e3:.3e} updates/s, launches {s.kernel_launches}", flush=True)
s.close()
