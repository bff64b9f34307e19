timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical sts:strassen:s sts_serp:strassen:s:LCMA_SERPENTINE=1 sts_swz4:strassen:s:LCMA_SWZ=4 sts_swz16:strassen:s:LCMA_SWZ=16 sts_swz4s:strassen:s:LCMA_SWZ=4,LCMA_SERPENTINE=1
LCMA_LIB=$PWD/paper_2605_06057_b200/liblcma_s5.so timeout 300 python tools/cmp.py 8192 14336 4096 cl5:classical sts5:strassen:s sts5_serp:strassen:s:LCMA_SERPENTINE=1
timeout 600 python tools/cmp.py 32768 28672 8192 cl:classical sts:strassen:s sts_serp:strassen:s:LCMA_SERPENTINE=1
