cd $GRAFT_REPO_ROOT
export LCMA_LIB=$GRAFT_REPO_ROOT/paper_2605_06057_b200/liblcma_diag.so
python tools/r02/epi_ablate.py 8192 14336 4096 > gpurun_out/r02n_ablate.txt 2>&1
python tools/r02/epi_ablate.py 32768 28672 8192 > gpurun_out/r02n_ablate5.txt 2>&1
