cd $GRAFT_REPO_ROOT
export BL=1 REPS=2 DT=0 LCMA_LIB=$PWD/paper_2605_06057_b200/liblcma_diag.so
ROUNDS=5 timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical sts1:strassen:s:LCMA_CST=1 sts0:strassen:s:LCMA_CST=0
ROUNDS=3 timeout 600 python tools/cmp.py 32768 28672 8192 cl:classical sts1:strassen:s:LCMA_CST=1 sts0:strassen:s:LCMA_CST=0 st0:strassen:LCMA_CST=0
ROUNDS=3 timeout 400 python tools/cmp.py 12288 12288 12288 cl:classical sts1:strassen:s:LCMA_CST=1 sts0:strassen:s:LCMA_CST=0
ROUNDS=3 timeout 400 python tools/cmp.py 16384 14336 4096 cl:classical sts1:strassen:s:LCMA_CST=1 sts0:strassen:s:LCMA_CST=0
