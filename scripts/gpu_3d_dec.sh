set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "3d or cfg5 or slab or basket" > gpurun_out/pytest_3d.log 2>&1; tail -15 gpurun_out/pytest_3d.log
python scripts/step_probe.py cfg5 1 0 512
python scripts/step_probe.py cfg5 1 2 512
