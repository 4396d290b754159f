ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2_K6.csv python scripts/prof_cfg2.py 6 8 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:quad1d -s 3 -c 1 -o gpurun_out/prof_quad1d_v1 python scripts/prof_cfg2.py 6 6 > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:spline_pass -s 3 -c 1 -o gpurun_out/prof_spline_v1 python scripts/prof_cfg2.py 6 6 > gpurun_out/ncu_full2.log 2>&1
ls -la gpurun_out
