cd $GRAFT_REPO_ROOT
for lib in paper_2605_06057_b200/liblcma.so tools/r02/lib_np6.so tools/r02/lib_np7.so; do
  echo "== $lib"
  LCMA_LIB=$lib ROUNDS=3 REPS=2 python tools/cmp.py 32768 28672 8192 classical:classical 2>&1 | tail -1
  LCMA_LIB=$lib ROUNDS=5 REPS=5 python tools/cmp.py 8192 14336 4096 classical:classical 2>&1 | tail -1
done
