# d >= 2 iteration: 2-D / 3-D parity tests, full-size step timings
set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "2d or 3d or cfg4 or cfg5 or slab or exchange or ex4 or heat" > gpurun_out/pytest_23.log 2>&1; tail -3 gpurun_out/pytest_23.log
python scripts/step_probe.py cfg4 3 0
python scripts/step_probe.py cfg5 1 0 512
python -c "
from paper_1909_13560_b200 import measure_fp64_peak
for i in range(3): print(measure_fp64_peak(0))"
