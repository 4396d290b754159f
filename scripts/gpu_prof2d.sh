ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4_step.csv python scripts/step_probe.py cfg4 2 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:quad2d -c 1 -o gpurun_out/prof_quad2d python scripts/step_probe.py cfg4 1 0 > gpurun_out/ncu2d.log 2>&1
tail -1 gpurun_out/ncu2d.log
python __graft_entry__.py --smoke 2>&1 | tail -3
