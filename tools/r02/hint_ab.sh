cd $GRAFT_REPO_ROOT
export BL=1 REPS=3 DT=0 LCMA_LIB=$PWD/paper_2605_06057_b200/liblcma_diag.so
ROUNDS=5 timeout 300 python tools/cmp.py 8192 14336 4096 sts:strassen:s h1:strassen:s:LCMA_OPERAND_HINT=1 h2:strassen:s:LCMA_OPERAND_HINT=2 h3:strassen:s:LCMA_OPERAND_HINT=3 h4:strassen:s:LCMA_OPERAND_HINT=4 sp:strassen:s:LCMA_SERPENTINE=1 cl:classical clh2:classical:LCMA_OPERAND_HINT=2
ROUNDS=3 REPS=2 timeout 900 python tools/cmp.py 32768 28672 8192 sts:strassen:s h2:strassen:s:LCMA_OPERAND_HINT=2 h3:strassen:s:LCMA_OPERAND_HINT=3 sp:strassen:s:LCMA_SERPENTINE=1 cl:classical
