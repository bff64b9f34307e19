timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical st:strassen sts:strassen:s s16:strassen:s:LCMA_DEBUG=16 s17:strassen:s:LCMA_DEBUG=17 cl16:classical:LCMA_DEBUG=16 sts_nosm:strassen:s:LCMA_SMEM_PARTIAL=0 stsqf:strassen:s:LCMA_QFULL=1
timeout 600 python tools/cmp.py 32768 28672 8192 cl:classical st:strassen sts:strassen:s
