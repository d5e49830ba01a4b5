python scripts/bwd_compare.py 0.05 16
python scripts/bwd_compare.py
CPDDG_ENVELOPE=sym python scripts/bwd_compare.py
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
