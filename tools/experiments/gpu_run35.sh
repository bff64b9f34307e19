timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "classical or random" 2>&1 | tail -1
for lib in "" np6 np7; do
  if [ -n "$lib" ]; then export LCMA_LIB=$PWD/paper_2605_06057_b200/liblcma_$lib.so; fi
  echo "== lib $lib"
  ROUNDS=5 timeout 600 python tools/cmp.py 32768 28672 8192 cl:classical cl8:classical:LCMA_SWZ=8
  ROUNDS=5 timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical
  ROUNDS=5 timeout 300 python tools/cmp.py 12288 12288 12288 cl:classical
done
