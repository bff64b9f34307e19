timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "producer" 2>&1 | tail -5
