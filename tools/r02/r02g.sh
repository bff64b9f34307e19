cd $GRAFT_REPO_ROOT
export LCMA_LIB=$GRAFT_REPO_ROOT/paper_2605_06057_b200/liblcma_diag.so
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/r02g_clocks.csv &
SMI=$!
export ROUNDS=7 REPS=5
python tools/cmp.py 8192 14336 4096 st:classical:sched=4:LCMA_PF=0 st_pf:classical:sched=4:LCMA_PF=1 dy:classical:LCMA_PF=0 dy_pf:classical:LCMA_PF=1 dy_pf8:classical:swz=8:LCMA_PF=1 > gpurun_out/r02g_cfg2_cls.txt 2>&1
python tools/cmp.py 8192 14336 4096 st:strassen:s:sched=4:LCMA_PF=0 st_pf:strassen:s:sched=4:LCMA_PF=1 dy:strassen:s:LCMA_PF=0 dy_pf:strassen:s:LCMA_PF=1 dy_pf4:strassen:s:swz=4:LCMA_PF=1 > gpurun_out/r02g_cfg2_str.txt 2>&1
export ROUNDS=5 REPS=2
python tools/cmp.py 32768 28672 8192 st:classical:sched=4:LCMA_PF=0 st_pf:classical:sched=4:LCMA_PF=1 dy:classical:LCMA_PF=0 dy_pf:classical:LCMA_PF=1 dy_pf8:classical:swz=8:LCMA_PF=1 > gpurun_out/r02g_cfg5_cls.txt 2>&1
python tools/cmp.py 32768 28672 8192 st:strassen:s:sched=4:LCMA_PF=0 st_pf:strassen:s:sched=4:LCMA_PF=1 dy:strassen:s:LCMA_PF=0 dy_pf:strassen:s:LCMA_PF=1 dy_pf4:strassen:s:swz=4:LCMA_PF=1 > gpurun_out/r02g_cfg5_str.txt 2>&1
kill $SMI
python tools/r02/kwait.py 8192 14336 4096 > gpurun_out/r02g_kwait_cfg2.txt 2>&1
