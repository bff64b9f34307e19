cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/s2_pytest.txt 2>&1; tail -2 gpurun_out/s2_pytest.txt
export BL=1 REPS=2 DT=0 ROUNDS=3
timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical s2:strassen2 s2f:strassen2:variant=fused_h s2s:strassen2:s s2fs:strassen2:s:variant=fused_h lad:laderman lads:laderman:s
timeout 600 python tools/cmp.py 12288 12288 12288 cl:classical s2:strassen2 s2f:strassen2:variant=fused_h s2s:strassen2:s s2fs:strassen2:s:variant=fused_h lads:laderman:s sts:strassen:s
