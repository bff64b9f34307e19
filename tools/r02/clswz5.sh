cd $GRAFT_REPO_ROOT
export BL=1 REPS=2 DT=0 ROUNDS=9
timeout 1200 python tools/cmp.py 32768 28672 8192 c8:classical:swz=8 c16:classical sts:strassen:s
