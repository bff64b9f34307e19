for i in 1 2; do
ROUNDS=7 timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical sts:strassen:s sts1:strassen:s:LCMA_DEBUG=1
ROUNDS=7 LCMA_LIB=$PWD/paper_2605_06057_b200/liblcma_p96.so timeout 300 python tools/cmp.py 8192 14336 4096 cl96:classical sts96:strassen:s
ROUNDS=7 LCMA_LIB=$PWD/paper_2605_06057_b200/liblcma_p64.so timeout 300 python tools/cmp.py 8192 14336 4096 cl64:classical sts64:strassen:s
done
