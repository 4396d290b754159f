#!/bin/bash
# ncu evidence of round 2 (run under gpurun from the repo root; one GPU):
#   launch lists of the bench step and of full-size cfg 4 / cfg 5 steps, and --set full captures
#   of the dominant kernels, summarised on the box into gpurun_out/r2prof/*.json / *.csv by
#   scripts/ncu_summary.py (the .ncu-rep files stay on the box: gpurun returns <= 64 MiB)
OUT=gpurun_out/r2prof
mkdir -p $OUT /tmp/r2rep
NCU="ncu --clock-control none"
summ() {  # report, json, regex
  python scripts/ncu_summary.py /tmp/r2rep/$1.ncu-rep $OUT/$2 "$3" > /dev/null 2>> $OUT/summary_errors.log
}
# (1) launch list of the bench command (per-launch times are cold-cache and serialised)
$NCU --metrics gpu__time_duration.sum -c 200 --csv --log-file $OUT/launches_bench.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-tts --no-d23 > $OUT/bench_under_ncu.log 2>&1
# (2) the headline kernel: one batched launch (cfg 2, K = 1..6), summary + per-line source page
$NCU --set full --import-source on -k regex:quad1d_fused -c 1 -o /tmp/r2rep/batch python scripts/prof_batch.py > $OUT/p1.log 2>&1
summ batch ncu_quad1d_fused_batch_summary.json quad1d_fused
ncu -i /tmp/r2rep/batch.ncu-rep --page source --csv --print-source cuda,sass > /tmp/r2rep/src.csv 2>/dev/null
python scripts/ncu_lines.py /tmp/r2rep/src.csv 60 > $OUT/quad1d_fused_lines.txt 2>&1
# (3) cfg 4 full size: one step's launches, aff_rows and the two spline passes
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active \
    --csv --log-file $OUT/launches_cfg4_step.csv python scripts/step_probe.py cfg4 1 0 4096 > $OUT/p2.log 2>&1
$NCU --set full -k regex:aff_rows -c 1 -o /tmp/r2rep/aff python scripts/step_probe.py cfg4 1 0 4096 > $OUT/p3.log 2>&1
summ aff ncu_aff_rows_cfg4_summary.json aff_rows
$NCU --set full -k regex:spline_rf -s 6 -c 2 -o /tmp/r2rep/spl4 python scripts/step_probe.py cfg4 1 0 4096 > $OUT/p4.log 2>&1
summ spl4 ncu_spline_rf_strided_cfg4_summary.json "spline_rf<20, true>|spline_rf<20, 1>"
summ spl4 ncu_spline_rf_contig_cfg4_summary.json "spline_rf<20, false>|spline_rf<20, 0>"
# (4) cfg 5 full size (512^3): the decomposed path's quad3d and the spline passes
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active \
    --csv --log-file $OUT/launches_cfg5_step.csv python scripts/step_probe.py cfg5 1 0 512 > $OUT/p5.log 2>&1
$NCU --set full -k regex:quad3d -c 1 -o /tmp/r2rep/q3 python scripts/step_probe.py cfg5 1 0 512 > $OUT/p6.log 2>&1
summ q3 ncu_quad3d_dec_cfg5_summary.json quad3d
$NCU --set full -k regex:spline_rf -s 12 -c 3 -o /tmp/r2rep/spl5 python scripts/step_probe.py cfg5 1 0 512 > $OUT/p7.log 2>&1
summ spl5 ncu_spline_rf_strided_cfg5_summary.json "spline_rf<20, true>|spline_rf<20, 1>"
summ spl5 ncu_spline_rf_contig_cfg5_summary.json "spline_rf<20, false>|spline_rf<20, 0>"
ls -la $OUT
