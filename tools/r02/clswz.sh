cd $GRAFT_REPO_ROOT
export BL=1 REPS=3 DT=0 ROUNDS=5
timeout 300 python tools/cmp.py 8192 14336 4096 c16:classical c8:classical:swz=8 c32:classical:swz=32 c4:classical:swz=4
ROUNDS=3 REPS=2 timeout 900 python tools/cmp.py 32768 28672 8192 c16:classical c8:classical:swz=8 c32:classical:swz=32
