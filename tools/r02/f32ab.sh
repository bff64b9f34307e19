cd $GRAFT_REPO_ROOT
export BL=0 REPS=2 ROUNDS=5
for lib in "" "$PWD/tools/r02/lib_f32single.so" "" "$PWD/tools/r02/lib_f32single.so"; do
  echo "== ${lib:-current}"
  LCMA_LIB=$lib DT=2 timeout 300 python tools/cmp.py 16384 14336 14336 cl:classical st:strassen | tail -1
  LCMA_LIB=$lib DT=0 BL=1 timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical s2:strassen2 | tail -1
done
