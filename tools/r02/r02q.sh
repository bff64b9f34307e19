cd $GRAFT_REPO_ROOT
export LCMA_LIB=$GRAFT_REPO_ROOT/paper_2605_06057_b200/liblcma_diag.so
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv -lms 100 > gpurun_out/r02q_smi.csv &
SMI=$!
python tools/r02/epi_ablate.py 8192 14336 4096 > gpurun_out/r02q_ablate.txt 2>&1
kill $SMI
