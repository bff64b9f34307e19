ROUNDS=5 timeout 900 python tools/cmp.py 12288 12288 12288 cl16:classical cl8:classical:LCMA_SWZ=8 cl4:classical:LCMA_SWZ=4 sts8:strassen:s sts4:strassen:s:LCMA_SWZ=4
ROUNDS=5 timeout 900 python tools/cmp.py 16384 4096 14336 cl16:classical cl8:classical:LCMA_SWZ=8 cl4:classical:LCMA_SWZ=4
ROUNDS=5 timeout 900 python tools/cmp.py 16384 14336 4096 cl16:classical cl8:classical:LCMA_SWZ=8 cl4:classical:LCMA_SWZ=4
ROUNDS=5 timeout 900 python tools/cmp.py 16384 28672 8192 cl16:classical cl8:classical:LCMA_SWZ=8 cl4:classical:LCMA_SWZ=4 sts8:strassen:s
