# one GPU session: tests, bench, launch list, ncu capture of the hot kernel
set -x
nproc; lscpu | grep "Model name"
python __graft_entry__.py --smoke 2>&1 | tail -3
timeout 1500 python -m pytest tests/ -m gpu -q --durations=20 -x 2>&1 | tail -40
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2_K6.csv python scripts/prof_cfg2.py 6 8 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:quad1d_fused -s 3 -c 1 -o gpurun_out/prof_quad1d_fused python scripts/prof_cfg2.py 6 6 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
