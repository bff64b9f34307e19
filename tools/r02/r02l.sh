cd $GRAFT_REPO_ROOT
export ROUNDS=7 REPS=5
python tools/cmp.py 8192 14336 4096 cls:classical str:strassen sst:strassen:s cls_d:classical:sched=5 sst_d:strassen:s:sched=5 > gpurun_out/r02l_cfg2.txt 2>&1
export LCMA_LIB=$GRAFT_REPO_ROOT/paper_2605_06057_b200/liblcma_diag.so
python tools/r02/epi_ablate.py 8192 14336 4096 > gpurun_out/r02l_ablate.txt 2>&1
