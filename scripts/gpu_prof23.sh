# ncu --set full (with source) of one quad2d launch (cfg 4) and one quad3d launch (cfg 5 shape at 256^3)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:quad2d -c 1 -o gpurun_out/prof_quad2d_r1b python scripts/step_probe.py cfg4 1 0 > gpurun_out/ncu2d.log 2>&1
tail -1 gpurun_out/ncu2d.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:quad3d -c 1 -o gpurun_out/prof_quad3d_r1b python scripts/step_probe.py cfg5 1 0 256 > gpurun_out/ncu3d.log 2>&1
tail -1 gpurun_out/ncu3d.log
python scripts/step_probe.py cfg4 3 0
