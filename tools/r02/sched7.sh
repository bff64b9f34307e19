cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "dynamic_vs_static or split" > gpurun_out/s7_pytest.txt 2>&1; tail -3 gpurun_out/s7_pytest.txt
export BL=1 REPS=2 DT=0
ROUNDS=5 timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical cl5:classical:sched=5 sts:strassen:s sts7:strassen:s:sched=7 st:strassen st7:strassen:sched=7
ROUNDS=3 timeout 900 python tools/cmp.py 32768 28672 8192 cl:classical cl5:classical:sched=5 sts:strassen:s sts7:strassen:s:sched=7 st:strassen st7:strassen:sched=7
ROUNDS=3 timeout 600 python tools/cmp.py 12288 12288 12288 cl:classical cl5:classical:sched=5 sts:strassen:s sts7:strassen:s:sched=7
