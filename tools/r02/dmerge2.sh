cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/dmerge2_pytest.txt 2>&1; tail -15 gpurun_out/dmerge2_pytest.txt | grep -E "passed|failed|Error|FAILED|assert" | head
timeout 200 python tools/r02/tail.py 12288 12288 12288 strassen
export BL=1 REPS=2 DT=0
ROUNDS=5 timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical st:strassen sts:strassen:s
ROUNDS=3 timeout 600 python tools/cmp.py 32768 28672 8192 cl:classical st:strassen sts:strassen:s
ROUNDS=3 timeout 400 python tools/cmp.py 12288 12288 12288 cl:classical st:strassen sts:strassen:s
