timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do
ROUNDS=7 timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical sts:strassen:s sts1:strassen:s:LCMA_DEBUG=1 s1920:strassen:s:LCMA_DEBUG=1920
ROUNDS=7 LCMA_LIB=$PWD/paper_2605_06057_b200/liblcma_prev.so timeout 300 python tools/cmp.py 8192 14336 4096 clprev:classical stsprev:strassen:s sts1prev:strassen:s:LCMA_DEBUG=1 s1920prev:strassen:s:LCMA_DEBUG=1920
done
