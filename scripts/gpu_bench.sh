# bench + ncu evidence for the round (profiles are copied to profiles/ afterwards)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
timeout 300 python scripts/batch_time.py 0
timeout 300 python scripts/timeline2.py 10 1 6 2>&1 | tail -6
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 4000 gpurun_out/bench.json
tail -3 gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1; tail -c 1500 gpurun_out/bench_ref.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-tts --no-d23 > gpurun_out/bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:quad1d_fused -c 1 -o gpurun_out/prof_quad1d_fused_batch python scripts/prof_batch.py > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
