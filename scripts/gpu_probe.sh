#!/bin/bash
# one-off profiling session: phase timeline of the fused 1-D kernel (debug build), source-line
# ncu captures of quad3d and spline_pass (summaries into gpurun_out/probe)
OUT=gpurun_out/probe
mkdir -p $OUT /tmp/prep
for K in 6 3 1; do BSDE_PHASE_TIMING=1 timeout 300 python scripts/phase_timeline.py $K 0 293 > $OUT/phase_K$K.txt 2>&1; done
timeout 300 python scripts/step_probe.py cfg5 2 0 256 > $OUT/cfg5_256.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:quad3d -c 1 -o /tmp/prep/q3 python scripts/step_probe.py cfg5 1 0 256 > $OUT/n1.log 2>&1
ncu -i /tmp/prep/q3.ncu-rep --page source --csv --print-source cuda,sass > /tmp/prep/q3src.csv 2>/dev/null
python scripts/ncu_lines.py /tmp/prep/q3src.csv 50 > $OUT/quad3d_lines.txt 2>&1
python scripts/ncu_summary.py /tmp/prep/q3.ncu-rep $OUT/quad3d_summary.json quad3d > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:spline_pass -s 8 -c 2 -o /tmp/prep/spl python scripts/step_probe.py cfg4 1 0 4096 > $OUT/n2.log 2>&1
ncu -i /tmp/prep/spl.ncu-rep --page source --csv --print-source cuda,sass > /tmp/prep/splsrc.csv 2>/dev/null
python scripts/ncu_lines.py /tmp/prep/splsrc.csv 40 > $OUT/spline_lines.txt 2>&1
ncu -i /tmp/prep/spl.ncu-rep --page raw --csv > $OUT/spline_raw.csv 2>/dev/null
ls -la $OUT
