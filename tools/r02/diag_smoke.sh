cd $GRAFT_REPO_ROOT
export BL=1 ROUNDS=1 REPS=1 DT=0
D=$PWD/paper_2605_06057_b200/liblcma_diag.so
for arm in "cl:classical" "sts:strassen:s" "d1:strassen:s:LCMA_DEBUG=1" "d16:strassen:s:LCMA_DEBUG=16"; do
  echo "== $arm"; LCMA_LIB=$D timeout 60 python tools/cmp.py 8192 14336 4096 $arm 2>&1 | tail -2; echo "rc=$?"
done
echo "== product sts"; timeout 60 python tools/cmp.py 8192 14336 4096 sts:strassen:s 2>&1 | tail -2
