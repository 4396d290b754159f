#!/bin/bash
# ncu evidence of round 2 (run under gpurun from the repo root; one GPU):
#   launch lists of the bench step and of full-size cfg 4 / cfg 5 steps, and --set full captures
#   of the dominant kernels, summarised into profiles/round2/*.json by scripts/ncu_summary.py
set -x
OUT=gpurun_out/r2prof
mkdir -p $OUT
NCU="ncu --clock-control none"
# (1) launch list of the bench command (its per-launch times are cold-cache and serialised)
$NCU --metrics gpu__time_duration.sum -c 200 --csv --log-file $OUT/launches_bench.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-tts --no-d23 > $OUT/bench_under_ncu.log 2>&1
# (2) the headline kernel: one batched launch (cfg 2, K = 1..6)
$NCU --set full --import-source on -k regex:quad1d_fused -c 1 -o $OUT/prof_batch python scripts/prof_batch.py > $OUT/p1.log 2>&1
# (3) cfg 4 full size: one step's kernels (aff_axis0, aff_rows, spline passes)
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active \
    --csv --log-file $OUT/launches_cfg4_step.csv python scripts/step_probe.py cfg4 1 0 4096 > $OUT/p2.log 2>&1
$NCU --set full -k regex:aff_rows -c 1 -o $OUT/prof_aff_rows_cfg4 python scripts/step_probe.py cfg4 1 0 4096 > $OUT/p3.log 2>&1
$NCU --set full -k regex:spline_pass -s 3 -c 2 -o $OUT/prof_spline_cfg4 python scripts/step_probe.py cfg4 1 0 4096 > $OUT/p4.log 2>&1
# (4) cfg 5 full size (512^3): the decomposed path's quad3d and a strided / contiguous spline pass
$NCU --set full -k regex:quad3d -c 1 -o $OUT/prof_quad3d_cfg5 python scripts/step_probe.py cfg5 1 0 512 > $OUT/p5.log 2>&1
$NCU --set full -k regex:spline_pass -s 12 -c 3 -o $OUT/prof_spline_cfg5 python scripts/step_probe.py cfg5 1 0 512 > $OUT/p6.log 2>&1
ls -la $OUT
