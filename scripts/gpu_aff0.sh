set -x
python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; tail -4 gpurun_out/smoke.log
python scripts/step_probe.py cfg4 3 0
BSDE_AFF0_STAGED=1 python scripts/step_probe.py cfg4 3 0
BSDE_AFF0_STAGED=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "2d or cfg4 or exchange or ex4 or heat" > gpurun_out/pytest_aff0.log 2>&1; tail -2 gpurun_out/pytest_aff0.log
