cd $GRAFT_REPO_ROOT
export BL=1 ROUNDS=5 REPS=3 LCMA_LIB=$PWD/paper_2605_06057_b200/liblcma_diag.so
DT=4 timeout 300 python tools/cmp.py 8192 14336 4096 cls:classical:s nosf:classical:s:LCMA_DEBUG=4096 nocp:classical:s:LCMA_DEBUG=8192 nosfcp:classical:s:LCMA_DEBUG=12288 noload:classical:s:LCMA_DEBUG=16 noepi:classical:s:LCMA_DEBUG=1
DT=0 timeout 300 python tools/cmp.py 8192 14336 4096 b256:classical b128:classical:LCMA_BN=128 b128noload:classical:LCMA_BN=128,LCMA_DEBUG=16 b256noload:classical:LCMA_DEBUG=16
