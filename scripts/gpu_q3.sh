#!/bin/bash
# quad3d iteration: 3-D parity tests, cfg 5 step time (512^3), ncu of quad3d at 256^3
OUT=gpurun_out/q3; mkdir -p $OUT /tmp/q3
timeout 900 python -m pytest tests -m gpu -x -q -k "3d or cfg5 or basket" > $OUT/tests.log 2>&1; echo rc=$? >> $OUT/tests.log
timeout 300 python scripts/step_probe.py cfg5 2 0 512 > $OUT/cfg5.txt 2>&1
timeout 300 python scripts/step_probe.py cfg4 3 0 4096 > $OUT/cfg4.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:quad3d -c 1 -o /tmp/q3/q3 python scripts/step_probe.py cfg5 1 0 256 > $OUT/n1.log 2>&1
ncu -i /tmp/q3/q3.ncu-rep --page source --csv --print-source cuda,sass > /tmp/q3/src.csv 2>/dev/null
python scripts/ncu_lines.py /tmp/q3/src.csv 40 > $OUT/quad3d_lines.txt 2>&1
python scripts/ncu_summary.py /tmp/q3/q3.ncu-rep $OUT/quad3d_summary.json quad3d > /dev/null 2>&1
