cd $GRAFT_REPO_ROOT
export BL=1 REPS=3 DT=0 LCMA_LIB=$PWD/paper_2605_06057_b200/liblcma_diag.so
ROUNDS=7 timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical st:strassen st0:strassen:LCMA_DIRECT=0 sts:strassen:s sts0:strassen:s:LCMA_DIRECT=0
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 300 ncu --metrics $M --clock-control none -k regex:group_combine -c 2 python tools/ncu_one.py strassen x 8192 14336 4096 2>&1 | grep -E "group_comb|duration|dram"
