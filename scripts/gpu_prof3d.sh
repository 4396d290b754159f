ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5_step.csv python scripts/step_probe.py cfg5 1 0 512 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:quad3d -c 1 -o gpurun_out/prof_quad3d python scripts/step_probe.py cfg5 1 0 256 > gpurun_out/ncu3d.log 2>&1
tail -2 gpurun_out/ncu3d.log
