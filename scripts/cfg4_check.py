import sys
sys.path.insert(0, ".")
import torch, numpy as np
from paper_1909_13560_b200 import Solver, workloads as W
P = int(sys.argv[1])
s = Solver(W.cfg4(P))
print("level", s.level, flush=True)
s.step()
torch.cuda.synchronize()
y = s.layer(0)
print("ok step, y range", float(y.min()), float(y.max()), flush=True)
