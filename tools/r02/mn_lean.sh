cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/mn_pytest.txt 2>&1; tail -2 gpurun_out/mn_pytest.txt
export REPS=3 ROUNDS=5
BL=0 DT=1 timeout 300 python tools/cmp.py 12288 14336 14336 cl:classical st:strassen
BL=0 DT=0 timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical st:strassen
BL=1 DT=0 timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical st:strassen
BL=0 DT=2 timeout 300 python tools/cmp.py 16384 14336 14336 cl:classical st:strassen
