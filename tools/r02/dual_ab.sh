cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/dual_pytest.txt 2>&1; tail -2 gpurun_out/dual_pytest.txt
export BL=1 REPS=3 DT=0 LCMA_LIB=$PWD/paper_2605_06057_b200/liblcma_diag.so
ROUNDS=7 timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical st:strassen sp:strassen:LCMA_COMB_SPLIT=1 s2:strassen2 s2p:strassen2:LCMA_COMB_SPLIT=1
ROUNDS=3 REPS=2 timeout 900 python tools/cmp.py 32768 28672 8192 cl:classical st:strassen sp:strassen:LCMA_COMB_SPLIT=1
