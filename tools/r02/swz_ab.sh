cd $GRAFT_REPO_ROOT
export BL=1 REPS=2 DT=0
ROUNDS=5 timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical s8:strassen:s s4:strassen:s:swz=4 s2:strassen:s:swz=2 s16:strassen:s:swz=16 s6:strassen:s:swz=6
ROUNDS=3 timeout 900 python tools/cmp.py 32768 28672 8192 cl:classical s8:strassen:s s4:strassen:s:swz=4 s16:strassen:s:swz=16 s12:strassen:s:swz=12
