#!/bin/bash
# spline iteration: d >= 2 parity tests, cfg 4 / cfg 5 step times, launch list of a cfg 4 step
OUT=gpurun_out/spl; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q -k "2d or 3d or cfg4 or cfg5 or slab or spline or heat or constant or fd_bicubic or fsde or printed" --deselect tests/test_gpu_parity.py::test_cfg4_full_solve_1025 > $OUT/tests.log 2>&1; echo rc=$? >> $OUT/tests.log
timeout 300 python scripts/step_probe.py cfg4 3 0 4096 > $OUT/cfg4.txt 2>&1
timeout 300 python scripts/step_probe.py cfg5 2 0 512 > $OUT/cfg5.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches_cfg4.csv python scripts/step_probe.py cfg4 1 0 4096 > $OUT/n1.log 2>&1
