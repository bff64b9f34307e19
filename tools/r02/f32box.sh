cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/f32b_pytest.txt 2>&1; tail -1 gpurun_out/f32b_pytest.txt
export BL=1 REPS=2 DT=0 ROUNDS=5
timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical s2:strassen2 s2s:strassen2:s
ROUNDS=3 timeout 600 python tools/cmp.py 12288 12288 12288 cl:classical s2s:strassen2:s
BL=0 DT=2 ROUNDS=3 timeout 300 python tools/cmp.py 16384 14336 14336 cl:classical st:strassen
