cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/ctma_pytest.txt 2>&1; tail -3 gpurun_out/ctma_pytest.txt
export BL=1 ROUNDS=5 REPS=3 DT=0
timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical st:strassen sts:strassen:s
LCMA_LIB=$PWD/paper_2605_06057_b200/liblcma_diag.so timeout 300 python tools/cmp.py 8192 14336 4096 sts:strassen:s sts_notma:strassen:s:LCMA_C_TMA=0 cl:classical cl_notma:classical:LCMA_C_TMA=0
DT=4 timeout 300 python tools/cmp.py 8192 14336 4096 cls:classical:s sts:strassen:s
timeout 120 python tools/timeline.py strassen 8192 14336 4096
ROUNDS=3 timeout 600 python tools/cmp.py 32768 28672 8192 cl:classical st:strassen sts:strassen:s
