#!/bin/bash
OUT=gpurun_out/spl; mkdir -p $OUT
timeout 300 python scripts/step_probe.py cfg4 3 0 4096 > $OUT/cfg4.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches_cfg4.csv python scripts/step_probe.py cfg4 1 0 4096 > $OUT/n1.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "2d or 3d or slab or spline" > $OUT/tests.log 2>&1; echo rc=$? >> $OUT/tests.log
