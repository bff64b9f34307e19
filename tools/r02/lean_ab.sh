cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/lean_pytest.txt 2>&1; tail -2 gpurun_out/lean_pytest.txt
export BL=1 ROUNDS=5 REPS=3
D=$PWD/paper_2605_06057_b200/liblcma_diag.so
for lib in "" $D ""; do
  echo "== LIB ${lib:-product}"
  LCMA_LIB=$lib DT=0 timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical st:strassen sts:strassen:s
  LCMA_LIB=$lib DT=4 timeout 300 python tools/cmp.py 8192 14336 4096 cls:classical:s sts:strassen:s
done
echo "== cfg5"
for lib in "" $D; do
  echo "== LIB ${lib:-product}"
  LCMA_LIB=$lib DT=0 ROUNDS=3 timeout 600 python tools/cmp.py 32768 28672 8192 cl:classical st:strassen sts:strassen:s
done
