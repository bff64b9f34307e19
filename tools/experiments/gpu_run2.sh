nvidia-smi --query-gpu=name,clocks.sm,power.draw --format=csv
S=8192\ 14336\ 4096
timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical st:strassen sts:strassen:s sts_ml:strassen:s:LCMA_DEBUG=1 cl_ml:classical:LCMA_DEBUG=1 sts_noreg:strassen:s:LCMA_REG_PARTIAL=0
timeout 600 python tools/cmp.py 32768 28672 8192 cl:classical st:strassen sts:strassen:s sts_ml:strassen:s:LCMA_DEBUG=1
ROUNDS=5 timeout 600 python tools/cmp.py 12288 12288 12288 cl:classical st:strassen lad:laderman s2:strassen2
