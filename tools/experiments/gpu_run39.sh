timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "producer" 2>&1 | tail -3
ROUNDS=5 timeout 600 python tools/cmp.py 8192 14336 4096 cl:classical st:strassen pf2:strassen:variant=producer pf1:strassen:variant=producer:LCMA_PF_A_ONLY=1
