cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x -k "dynamic or exact or determinism or graph" 2>&1 | tail -4 > gpurun_out/r02j_pytest.txt
export LCMA_LIB=$GRAFT_REPO_ROOT/paper_2605_06057_b200/liblcma_diag.so
export ROUNDS=9 REPS=5
python tools/cmp.py 8192 14336 4096 st:classical:sched=4:LCMA_PF=0 dy:classical:LCMA_PF=0 dy_pf:classical:LCMA_PF=1 sst:strassen:s:sched=4:LCMA_PF=0 sdy:strassen:s:LCMA_PF=0 sdy_pf:strassen:s:LCMA_PF=1 > gpurun_out/r02j_cfg2.txt 2>&1
export ROUNDS=5 REPS=2
python tools/cmp.py 32768 28672 8192 st:classical:sched=4:LCMA_PF=0 dy:classical:LCMA_PF=0 dy8:classical:swz=8:LCMA_PF=0 sst:strassen:s:sched=4:LCMA_PF=0 sdy:strassen:s:LCMA_PF=0 sdy4:strassen:s:swz=4:LCMA_PF=0 > gpurun_out/r02j_cfg5.txt 2>&1
python tools/r02/kwait.py 8192 14336 4096 > gpurun_out/r02j_kwait_cfg2.txt 2>&1
