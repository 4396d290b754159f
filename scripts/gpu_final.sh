# final round-1 session: smoke, full GPU suite, bench line, cfg 5 launch list, ncu of quad3d<DIFF,1>
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; tail -4 gpurun_out/smoke.log
timeout 1800 python -m pytest tests/ -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 600 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
bash scripts/gpu_3d_prof.sh > gpurun_out/cfg5_launches.txt 2>&1; cat gpurun_out/cfg5_launches.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:quad3d -c 1 -o gpurun_out/prof_quad3d_dec python scripts/step_probe.py cfg5 1 0 256 > gpurun_out/ncu3d.log 2>&1; tail -1 gpurun_out/ncu3d.log
python scripts/ncu_summary.py gpurun_out/prof_quad3d_dec.ncu-rep gpurun_out/ncu_quad3d_dec_cfg5_P256_summary.json quad3d
