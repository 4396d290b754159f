# 1-D diagnosis: phase timeline of the batched launch, fused variants, ncu --set full of the launch
set -x
python scripts/timeline_batch.py > gpurun_out/timeline.txt 2>&1; cat gpurun_out/timeline.txt
python scripts/batch_variants.py 0,1,2,3,4,5 > gpurun_out/variants.txt 2>&1; cat gpurun_out/variants.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:quad1d_fused -c 1 -o gpurun_out/prof_batch_r1b python scripts/prof_batch.py > gpurun_out/ncu_batch.log 2>&1; tail -3 gpurun_out/ncu_batch.log
