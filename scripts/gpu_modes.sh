timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
timeout 300 python scripts/batch_time.py 0
timeout 300 python scripts/timeline2.py 10 1 6 2>&1 | tail -6
timeout 300 python scripts/timeline_batch.py 2>&1 | head -8
