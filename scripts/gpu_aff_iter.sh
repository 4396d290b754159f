set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "2d or cfg4 or exchange or ex4 or heat or constant or slab or printed" > gpurun_out/pytest_aff.log 2>&1; tail -3 gpurun_out/pytest_aff.log
python scripts/step_probe.py cfg4 3 0
bash scripts/gpu_aff_prof.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:aff_rows -c 1 -o gpurun_out/prof_aff_rows_cfg4 python scripts/step_probe.py cfg4 1 0 > gpurun_out/ncu_affr.log 2>&1; tail -1 gpurun_out/ncu_affr.log
python scripts/ncu_summary.py gpurun_out/prof_aff_rows_cfg4.ncu-rep gpurun_out/ncu_aff_rows_cfg4_summary.json aff_rows
