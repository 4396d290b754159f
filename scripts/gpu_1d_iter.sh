# 1-D iteration: fused-path parity tests, batched timing, busy-time probe
set -x
python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cfg2 or fused or batch or printed or persistent or bootstrap or ky" > gpurun_out/pytest_1d.log 2>&1; tail -5 gpurun_out/pytest_1d.log
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv,noheader; python scripts/busy_probe.py > gpurun_out/busy.txt 2>&1; head -3 gpurun_out/busy.txt; grep "K=6" gpurun_out/busy.txt
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu,power.draw,clocks_throttle_reasons.active --format=csv,noheader
