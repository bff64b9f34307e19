timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical sts:strassen:s sts1:strassen:s:LCMA_DEBUG=1 st:strassen sts896:strassen:s:LCMA_DEBUG=896
timeout 600 python tools/cmp.py 32768 28672 8192 cl:classical st:strassen sts:strassen:s
