cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/r02e_pytest.txt
export ROUNDS=5 REPS=2
python tools/cmp.py 32768 28672 8192 static:classical:sched=4 d4:classical:swz=4 d6:classical:swz=6 d8:classical:swz=8 d12:classical:swz=12 > gpurun_out/r02e_cfg5_cls.txt 2>&1
python tools/cmp.py 32768 28672 8192 static:strassen:s:sched=4 d2:strassen:s:swz=2 d3:strassen:s:swz=3 d4:strassen:s:swz=4 d6:strassen:s:swz=6 > gpurun_out/r02e_cfg5_str.txt 2>&1
export ROUNDS=7 REPS=5
python tools/cmp.py 8192 14336 4096 static:classical:sched=4 d4:classical:swz=4 d8:classical:swz=8 d16:classical:swz=16 sstatic:strassen:s:sched=4 s2:strassen:s:swz=2 s4:strassen:s:swz=4 s8:strassen:s:swz=8 > gpurun_out/r02e_cfg2.txt 2>&1
