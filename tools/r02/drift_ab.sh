cd $GRAFT_REPO_ROOT
export BL=1 REPS=2 DT=0 LCMA_LIB=$PWD/paper_2605_06057_b200/liblcma_diag.so
ROUNDS=3 timeout 900 python tools/cmp.py 32768 28672 8192 cl:classical sts:strassen:s d1:strassen:s:LCMA_DRIFT=1 d2:strassen:s:LCMA_DRIFT=2 d4:strassen:s:LCMA_DRIFT=4 cls1:classical:sched=1 cls1d2:classical:sched=1:LCMA_DRIFT=2
ROUNDS=5 REPS=3 timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical sts:strassen:s d1:strassen:s:LCMA_DRIFT=1 d2:strassen:s:LCMA_DRIFT=2 d4:strassen:s:LCMA_DRIFT=4
M="gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
LCMA_DRIFT=2 timeout 900 ncu --metrics $M --clock-control none -k regex:umma -s 1 -c 1 python tools/ncu_one.py strassen static 32768 28672 8192 2>&1 | grep -E "duration|dram|hit|tensor"
