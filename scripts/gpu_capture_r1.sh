# round-1 evidence: bench line, reference arm, launch list of the bench, ncu --set full of the
# dominant kernels (quad1d_fused batch, aff_rows / aff_axis0 for cfg 4)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 1500 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-tts --no-d23 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:quad1d_fused -c 1 -o gpurun_out/prof_quad1d_batch_r1c python scripts/prof_batch.py > gpurun_out/ncu_b.log 2>&1; tail -1 gpurun_out/ncu_b.log
python scripts/ncu_summary.py gpurun_out/prof_quad1d_batch_r1c.ncu-rep gpurun_out/ncu_quad1d_fused_batch_summary.json quad1d
timeout 900 ncu --set full --clock-control none --import-source on -k regex:aff_ -c 2 -o gpurun_out/prof_aff2_cfg4 python scripts/step_probe.py cfg4 1 0 > gpurun_out/ncu_aff.log 2>&1; tail -1 gpurun_out/ncu_aff.log
python scripts/ncu_summary.py gpurun_out/prof_aff2_cfg4.ncu-rep gpurun_out/ncu_aff_axis0_cfg4_summary.json aff_axis0
python scripts/ncu_summary.py gpurun_out/prof_aff2_cfg4.ncu-rep gpurun_out/ncu_aff_rows_cfg4_summary.json aff_rows
bash scripts/gpu_aff_prof.sh
ls -la gpurun_out
