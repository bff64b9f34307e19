cd $GRAFT_REPO_ROOT
export BL=1 REPS=3 DT=0 LCMA_LIB=$PWD/paper_2605_06057_b200/liblcma_diag.so
ROUNDS=5 timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical sts:strassen:s a20:strassen:s:LCMA_L2PERSIST_A=20 a40:strassen:s:LCMA_L2PERSIST_A=40 a60:strassen:s:LCMA_L2PERSIST_A=60
ROUNDS=3 REPS=2 timeout 900 python tools/cmp.py 32768 28672 8192 cl:classical sts:strassen:s a40:strassen:s:LCMA_L2PERSIST_A=40
