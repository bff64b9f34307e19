cd $GRAFT_REPO_ROOT
export BL=1 REPS=3 DT=0 LCMA_LIB=$PWD/paper_2605_06057_b200/liblcma_diag.so
ROUNDS=7 timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical sts:strassen:s cs:strassen:s:LCMA_C_CS=1 ph0:strassen:s:LCMA_PARTIAL_HINT=0 csph0:strassen:s:LCMA_C_CS=1,LCMA_PARTIAL_HINT=0 clcs:classical:LCMA_C_CS=1
ROUNDS=3 REPS=2 timeout 900 python tools/cmp.py 32768 28672 8192 cl:classical sts:strassen:s cs:strassen:s:LCMA_C_CS=1 ph0:strassen:s:LCMA_PARTIAL_HINT=0 clcs:classical:LCMA_C_CS=1
