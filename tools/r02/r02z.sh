cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x --timeout 200 -k "strassen2 or two_level or diag_build or cfg4" -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/r02z_pytest.txt
export ROUNDS=7 REPS=5
timeout 600 python tools/cmp.py 8192 14336 4096 cls:classical s2:strassen2 s2s:strassen2:s > gpurun_out/r02z_cfg2.txt 2>&1
export ROUNDS=5 REPS=2
timeout 600 python tools/cmp.py 12288 12288 12288 cls:classical s2:strassen2 s2s:strassen2:s lad:laderman lads:laderman:s str:strassen strs:strassen:s > gpurun_out/r02z_cfg4.txt 2>&1
