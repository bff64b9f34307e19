cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/f32_pytest.txt 2>&1; tail -2 gpurun_out/f32_pytest.txt
export BL=1 REPS=2 DT=0 ROUNDS=3 LCMA_LIB=$PWD/paper_2605_06057_b200/liblcma_diag.so
timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical s2:strassen2 s2n:strassen2:LCMA_C_TMA=0 s2s:strassen2:s s2sn:strassen2:s:LCMA_C_TMA=0
timeout 600 python tools/cmp.py 12288 12288 12288 cl:classical s2:strassen2 s2n:strassen2:LCMA_C_TMA=0 s2s:strassen2:s
DT=2 timeout 300 python tools/cmp.py 16384 14336 14336 cl:classical st:strassen stn:strassen:LCMA_C_TMA=0
