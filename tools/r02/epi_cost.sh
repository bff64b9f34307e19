cd $GRAFT_REPO_ROOT
export BL=1 ROUNDS=5 REPS=3 LCMA_LIB=$PWD/paper_2605_06057_b200/liblcma_diag.so DT=0
timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical sts:strassen:s d1:strassen:s:LCMA_DEBUG=1 d128:strassen:s:LCMA_DEBUG=128 d256:strassen:s:LCMA_DEBUG=256 d512:strassen:s:LCMA_DEBUG=512 d1024:strassen:s:LCMA_DEBUG=1024 d1920:strassen:s:LCMA_DEBUG=1920
