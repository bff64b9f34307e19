cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -k "exact or tolerance or determinism or cfg2" 2>&1 | tail -3 > gpurun_out/r02m_pytest.txt
export ROUNDS=7 REPS=5
python tools/cmp.py 8192 14336 4096 cls:classical str:strassen sst:strassen:s > gpurun_out/r02m_cfg2.txt 2>&1
export ROUNDS=5 REPS=2
python tools/cmp.py 32768 28672 8192 cls:classical str:strassen sst:strassen:s > gpurun_out/r02m_cfg5.txt 2>&1
export LCMA_LIB=$GRAFT_REPO_ROOT/paper_2605_06057_b200/liblcma_diag.so
python tools/r02/epi_ablate.py 8192 14336 4096 > gpurun_out/r02m_ablate.txt 2>&1
