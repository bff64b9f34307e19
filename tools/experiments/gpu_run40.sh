timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
ROUNDS=5 timeout 600 python tools/cmp.py 8192 14336 4096 cl:classical st:strassen sts:strassen:s
