set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python __graft_entry__.py --smoke 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --durations=15 -k "not full_size" 2>&1 | tail -40
python - <<'PY'
import time
from paper_1909_13560_b200 import Solver, workloads as W
for K in [1,3,6]:
    for rep in range(2):
        with Solver(W.cfg2(K)) as s:
            r = s.solve()
            print(K, "sweep ms", r.t_sweep_s*1e3, "upd/s", r.updates/r.t_sweep_s, "y0", r.y0, "launches", s.kernel_launches)
PY
