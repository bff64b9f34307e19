cd $GRAFT_REPO_ROOT
export BL=1 REPS=3 DT=0 LCMA_LIB=$PWD/paper_2605_06057_b200/liblcma_diag.so
ROUNDS=5 timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical sts:strassen:s qf:strassen:s:LCMA_QFULL=1 d1:strassen:s:LCMA_DEBUG=1 d256:strassen:s:LCMA_DEBUG=256
ROUNDS=3 REPS=2 timeout 900 python tools/cmp.py 32768 28672 8192 cl:classical sts:strassen:s qf:strassen:s:LCMA_QFULL=1
