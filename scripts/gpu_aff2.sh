set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "2d or cfg4 or exchange or ex4 or heat or constant or slab or printed" > gpurun_out/pytest_aff.log 2>&1; tail -15 gpurun_out/pytest_aff.log
python scripts/step_probe.py cfg4 3 0
python scripts/step_probe.py cfg4 3 2
