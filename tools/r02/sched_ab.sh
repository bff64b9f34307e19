cd $GRAFT_REPO_ROOT
export BL=1 REPS=2 DT=0
ROUNDS=5 timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical sts:strassen:s sts5:strassen:s:sched=5 sts6:strassen:s:sched=6 cl5:classical:sched=5
ROUNDS=3 timeout 900 python tools/cmp.py 32768 28672 8192 cl:classical sts:strassen:s sts5:strassen:s:sched=5 sts6:strassen:s:sched=6 cl5:classical:sched=5
