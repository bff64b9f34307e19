ROUNDS=7 timeout 400 python tools/cmp.py 8192 14336 4096 cl:classical sts:strassen:s sts_er:strassen:s:LCMA_DEBUG=2048 sts1:strassen:s:LCMA_DEBUG=1 cl_er:classical:LCMA_DEBUG=2048
