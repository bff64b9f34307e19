cd $GRAFT_REPO_ROOT
timeout 700 python -m pytest tests/test_gpu_fp8.py -q > gpurun_out/fp8_tests3.txt 2>&1; grep -E "passed|failed|^FAILED" gpurun_out/fp8_tests3.txt | tail -8
export BL=1 ROUNDS=5 REPS=3
DT=4 timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical cls:classical:s st:strassen sts:strassen:s
DT=4 ROUNDS=3 timeout 600 python tools/cmp.py 32768 28672 8192 cl:classical cls:classical:s st:strassen sts:strassen:s
DT=4 timeout 200 python tools/cmp.py 2048 14336 4096 cl:classical cls:classical:s st:strassen sts:strassen:s
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
DT=4 timeout 600 ncu --metrics $M --clock-control none -k regex:"umma|combine" -c 3 python tools/ncu_one.py strassen x 8192 14336 4096 2>&1 | grep -E "umma|combine|duration|dram|tensor|hit"
