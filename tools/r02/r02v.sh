cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -k "dynamic" --timeout 120 2>&1 | tail -5 > gpurun_out/r02v_pytest.txt
export ROUNDS=9 REPS=5
timeout 600 python tools/cmp.py 8192 14336 4096 cls:classical cls6:classical:sched=6 sst:strassen:s sst6:strassen:s:sched=6 sst5:strassen:s:sched=5 > gpurun_out/r02v_cfg2.txt 2>&1
export ROUNDS=5 REPS=2
timeout 600 python tools/cmp.py 32768 28672 8192 cls:classical cls6:classical:sched=6 sst:strassen:s sst6:strassen:s:sched=6 > gpurun_out/r02v_cfg5.txt 2>&1
