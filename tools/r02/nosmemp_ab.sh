cd $GRAFT_REPO_ROOT
timeout 300 python tools/r02/nosmemp_check.py
export BL=1 REPS=2 DT=0 LCMA_LIB=$PWD/paper_2605_06057_b200/liblcma_diag.so
ROUNDS=7 timeout 1500 python tools/cmp.py 32768 28672 8192 cl:classical sts:strassen:s ns:strassen:s:LCMA_NOSMEMP=1
ROUNDS=5 timeout 600 python tools/cmp.py 12288 12288 12288 cl:classical sts:strassen:s ns:strassen:s:LCMA_NOSMEMP=1 lads:laderman:s lns:laderman:s:LCMA_NOSMEMP=1
