timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
ROUNDS=7 timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical sts:strassen:s
ROUNDS=7 LCMA_LIB=$PWD/paper_2605_06057_b200/liblcma_prev.so timeout 300 python tools/cmp.py 8192 14336 4096 clprev:classical stsprev:strassen:s
timeout 300 python tools/timeline.py strassen 32768 28672 8192
timeout 300 python tools/timeline.py classical 32768 28672 8192
