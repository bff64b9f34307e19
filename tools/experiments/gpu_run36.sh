timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "random or split" 2>&1 | tail -1
LCMA_SYNC=20 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "random or split" 2>&1 | tail -1
ROUNDS=5 timeout 900 python tools/cmp.py 32768 28672 8192 cl:classical cls:classical:LCMA_SYNC=20 cls8:classical:LCMA_SYNC=20,LCMA_SWZ=8 sts:strassen:s stss:strassen:s:LCMA_SYNC=20
ROUNDS=5 timeout 600 python tools/cmp.py 8192 14336 4096 cl:classical cls:classical:LCMA_SYNC=20 sts:strassen:s stss:strassen:s:LCMA_SYNC=20
