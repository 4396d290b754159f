"""Time a few backward steps of a BASELINE config at its full size (device events on a torch
stream).  usage: step_probe.py cfg4|cfg5 [steps] [kernel_variant] [P]"""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_1909_13560_b200 import Solver, workloads as W
name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
variant = int(sys.argv[3]) if len(sys.argv) > 3 else 0
P = int(sys.argv[4]) if len(sys.argv) > 4 else (4096 if name == "cfg4" else 512)
spec = W.cfg4(P) if name == "cfg4" else W.basket_3d(3, 64, 8, P=P)
ts = torch.cuda.Stream()
torch.cuda.set_stream(ts)
t0 = time.time()
s = Solver(spec, stream=ts.cuda_stream, kernel_variant=variant)
torch.cuda.synchronize()
print(f"{name} P={P} setup {time.time() - t0:.2f} s, shape {s.shape}", flush=True)
npts = 1
for n in s.shape:
    npts *= n
for rep in range(2):
    st = torch.cuda.Event(enable_timing=True)
    en = torch.cuda.Event(enable_timing=True)
    st.record(ts)
    for _ in range(steps):
        s.step()
    en.record(ts)
    torch.cuda.synchronize()
    ms = st.elapsed_time(en) / steps
    print(f"{name} P={P} variant={variant}: {ms:.3f} ms/step -> {npts / ms * 1e3:.3e} updates/s", flush=True)
s.close()
