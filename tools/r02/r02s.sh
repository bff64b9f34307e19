cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r02s_pytest.txt
export ROUNDS=7 REPS=5
python tools/cmp.py 8192 14336 4096 cls:classical str:strassen sst:strassen:s > gpurun_out/r02s_cfg2.txt 2>&1
