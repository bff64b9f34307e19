cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/dir_pytest.txt 2>&1; tail -15 gpurun_out/dir_pytest.txt | grep -E "passed|failed|Error|FAILED|assert" | head
export BL=1 REPS=3 DT=0 LCMA_LIB=$PWD/paper_2605_06057_b200/liblcma_diag.so
ROUNDS=5 timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical st:strassen st0:strassen:LCMA_DIRECT=0 sts:strassen:s sts0:strassen:s:LCMA_DIRECT=0
ROUNDS=3 REPS=2 timeout 600 python tools/cmp.py 32768 28672 8192 cl:classical st:strassen st0:strassen:LCMA_DIRECT=0 sts:strassen:s sts0:strassen:s:LCMA_DIRECT=0
