python scripts/phases2.py
python scripts/variants.py 5 2>&1
BSDE_NO_PERSISTENT=1 python scripts/variants.py 1 2>&1 | grep K=6
timeout 900 python -m pytest tests/ -m gpu -q -x 2>&1 | tail -4
