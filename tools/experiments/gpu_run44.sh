LCMA_L1PF=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "partial_homes or cfg2_bench or random" 2>&1 | tail -1
ROUNDS=7 timeout 400 python tools/cmp.py 8192 14336 4096 cl:classical sts:strassen:s stspf:strassen:s:LCMA_L1PF=1 st:strassen stpf:strassen:LCMA_L1PF=1
ROUNDS=5 timeout 600 python tools/cmp.py 32768 28672 8192 cl:classical sts:strassen:s stspf:strassen:s:LCMA_L1PF=1
