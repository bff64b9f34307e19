cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_fp8.py -q > gpurun_out/q8_tests.txt 2>&1; tail -1 gpurun_out/q8_tests.txt
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
DT=4 timeout 300 ncu --metrics $M --clock-control none -k regex:combine -c 2 python tools/ncu_one.py strassen x 8192 14336 4096 2>&1 | grep -E "q8|duration"
DT=4 timeout 300 ncu --metrics $M --clock-control none -k regex:combine -c 2 python tools/ncu_one.py classical x 8192 14336 4096 2>&1 | grep -E "q8|duration"
export BL=1 REPS=3 DT=4 ROUNDS=5
timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical st:strassen cls:classical:s sts:strassen:s
