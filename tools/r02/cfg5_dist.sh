cd $GRAFT_REPO_ROOT
export BL=1 REPS=2 DT=0 ROUNDS=15
timeout 1500 python tools/cmp.py 32768 28672 8192 cl:classical st:strassen sts:strassen:s
